"""Per-system iteration counts of one warm batched solve (C4 by default)."""
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
a = ap.parse_args()
cfg = CONFIGS[a.config]
ps = build_problem(cfg, device="cuda")
b = load_batch(Context(0), ps).tune_from_env()
bS = torch.tensor(ps.b_S, device="cuda")
for i in range(2):
    r = b.solve(bS, "dbj", 1e-10, 10 * cfg.max_iter, cfg.max_iter, "cgs2", True, history=False)
    torch.cuda.synchronize()
print("iterations", list(r.iterations))
