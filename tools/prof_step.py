"""One warm batched solve of a config (for ncu launch lists / captures)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1512_01756_b200 import Context  # noqa: E402
from paper_1512_01756_b200.configs import CONFIGS  # noqa: E402
from paper_1512_01756_b200.problems import build_problem, load_batch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--solves", type=int, default=2)
ap.add_argument("--orth", default="cgs2")
ap.add_argument("--modes", default="", help="subset of the config's systems, e.g. 1-12 (C5's slow low modes)")
ap.add_argument("--device-rhs", type=int, default=-1)
a = ap.parse_args()
cfg = CONFIGS[a.config]
modes = None
if a.modes:
    lo, _, hi = a.modes.partition("-")
    modes = list(range(int(lo), int(hi or lo) + 1))
drhs = cfg.k > 100_000 if a.device_rhs < 0 else bool(a.device_rhs)
ps = build_problem(cfg, modes, device="cuda", device_rhs=drhs, device_setup=drhs)
ctx = Context(0)
b = load_batch(ctx, ps).tune_from_env()
bS = torch.tensor(ps.b_S, device="cuda")
n0 = b.launch_count
for i in range(a.solves):
    r = b.solve(bS, "dbj", 1e-10, cfg.max_iter, 0, a.orth, True, history=False)
    torch.cuda.synchronize()
    print(f"solve {i}: launches {b.launch_count - n0} iterations max {max(r.iterations)} mean {sum(r.iterations)/len(r.iterations):.2f}", flush=True)
    n0 = b.launch_count
