"""b_S accuracy per mode: host FDM (numpy) vs device schur_rhs vs the oracle's
real-Schur shifted solve (the reference's route, proj/src/helmholtz.cpp:172-176)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_1512_01756_b200 import Context  # noqa: E402
from paper_1512_01756_b200.configs import CONFIGS  # noqa: E402
from paper_1512_01756_b200.problems import build_problem, load_batch, manufactured  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
check = [int(m) for m in (sys.argv[2] if len(sys.argv) > 2 else "1,37,40,41,42,43,55,86,87,88").split(",")]
host = build_problem(cfg, device="cuda")
dev = build_problem(cfg, device="cuda", device_rhs=True)
load_batch(Context(0), dev).tune_from_env()
rel = np.linalg.norm(dev.b_S - host.b_S, axis=1) / np.linalg.norm(host.b_S, axis=1)
order = np.argsort(-rel)
print("largest host/device b_S differences:", [(int(m), f"{rel[m]:.2e}") for m in order[:12]])
O.set_threads(8)
prob = O.Problem(cfg.n, cfg.m_x, cfg.m_z, cfg.l_x, cfg.l_z, cfg.c_tau)
for m in check:
    mu = host.mus[m]
    f, _ = manufactured(host.fdm.geo, cfg.kmax, cfg.decay, cfg.seed, m, mu=mu)
    ref = prob.apply_B(prob.shifted_solve(mu, f))
    nr = np.linalg.norm(ref)
    print(f"mode {m:3d} mu {mu:9.3f}: |ref| {nr:.3e} host-ref {np.linalg.norm(host.b_S[m] - ref) / nr:.2e} "
          f"dev-ref {np.linalg.norm(dev.b_S[m] - ref) / nr:.2e}", flush=True)
