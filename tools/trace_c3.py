"""One warm C3 solve with the tail traces on (SMPM_GT_TRACE / SMPM_GT_TRACE2 set by the caller)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1512_01756_b200 import Context  # noqa: E402
from paper_1512_01756_b200.configs import CONFIGS  # noqa: E402
from paper_1512_01756_b200.problems import build_problem, load_batch  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
ps = build_problem(cfg, device="cuda")
tr = {k: os.environ.pop(k) for k in ("SMPM_GT_TRACE", "SMPM_GT_TRACE2") if k in os.environ}
b = load_batch(Context(0), ps).tune_from_env()
bS = torch.tensor(ps.b_S, device="cuda")
for _ in range(2):
    b.solve(bS, "dbj", 1e-10, 10 * cfg.max_iter, cfg.max_iter, "cgs2", True, history=False)
for which, key in ((0, "SMPM_GT_TRACE"), (1, "SMPM_GT_TRACE2")):
    if key in tr:
        b.trace(which, tr[key])
r = b.solve(bS, "dbj", 1e-10, 10 * cfg.max_iter, cfg.max_iter, "cgs2", True, history=False)
torch.cuda.synchronize()
print("iterations", r.iterations)
