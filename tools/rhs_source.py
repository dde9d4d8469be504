"""Iteration counts of the C4 batch for three sources of the same b_S = B (A - mu)^{-1} f:
host FDM (numpy), device strip solver, and the oracle's real-Schur shifted solves (the
reference's route, proj/src/helmholtz.cpp:162-178)."""
import dataclasses
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_1512_01756_b200 import Context  # noqa: E402
from paper_1512_01756_b200.configs import CONFIGS  # noqa: E402
from paper_1512_01756_b200.fdm import project_out  # noqa: E402
from paper_1512_01756_b200.problems import build_problem, load_batch, manufactured  # noqa: E402

ctx = Context(0)
for sd in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "0,1,2").split(",")]:
    cfg = dataclasses.replace(CONFIGS["C4"], seed=1234 + sd)
    host = build_problem(cfg, device="cuda")
    dev = build_problem(cfg, device="cuda", device_rhs=True)
    b = load_batch(ctx, dev).tune_from_env()
    srcs = {"host": host.b_S, "device": dev.b_S}
    if sd == 0:
        O.set_threads(16)
        prob = O.Problem(cfg.n, cfg.m_x, cfg.m_z, cfg.l_x, cfg.l_z, cfg.c_tau)
        ob = []
        for m, mu in enumerate(host.mus):
            f, _ = manufactured(host.fdm.geo, cfg.kmax, cfg.decay, cfg.seed, m, mu=mu)
            if mu == 0.0:
                s0 = O.System(prob, 0.0, False)
                f = project_out(f, host.u_L)
                ob.append(project_out(s0.schur_rhs(f), host.u_S))
            else:
                ob.append(prob.apply_B(prob.shifted_solve(mu, f)))
        srcs["oracle"] = np.array(ob)
    for name, bs in srcs.items():
        r = b.solve(torch.tensor(bs, device="cuda"), "dbj", 1e-10, 1000, 100, "cgs2", True, history=False)
        print(f"seed {cfg.seed} {name:7s} iters sum {sum(r.iterations)} max {max(r.iterations)}", flush=True)
