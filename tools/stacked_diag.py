"""Stacked C4 subset: GPU vs oracle residual histories side by side."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_1512_01756_b200 import Context  # noqa: E402
from paper_1512_01756_b200.configs import CONFIGS  # noqa: E402
from paper_1512_01756_b200.problems import build_problem, load_batch  # noqa: E402

cfg = CONFIGS["C4"]
modes = [int(m) for m in (sys.argv[1] if len(sys.argv) > 1 else "0,1,2,5,37,127").split(",")]
ps = build_problem(cfg, modes, device="cuda")
b = load_batch(Context(0), ps).tune_from_env()
O.set_threads(8)
prob = O.Problem(cfg.n, cfg.m_x, cfg.m_z, cfg.l_x, cfg.l_z, cfg.c_tau)
systems = []
for i, mu in enumerate(ps.mus):
    s = O.System(prob, mu, False, kinds=(ps.GW[i], ps.GI[i], ps.GE[i]))
    s.build_bj(1)
    s.build_coarse(ps.u_S if mu == 0.0 else None)
    systems.append(s)
res = b.solve_stacked(torch.tensor(ps.b_S, device="cuda"), "dbj", 1e-10, 100)
ref = O.solve_stacked(systems, ps.b_S, "dbj", 1e-10, 100)
h, r = res.histories[0], ref.history
print("its", res.iterations[0], ref.iterations)
for i in range(max(len(h), len(r))):
    a = h[i] if i < len(h) else float("nan")
    c = r[i] if i < len(r) else float("nan")
    print(f"{i:3d} gpu {a:.6e} ref {c:.6e} rel {abs(a - c) / max(c, 1e-300):.2e}")
