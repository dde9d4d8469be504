"""Time warm C4 batched solves under different SMPM_* environment settings
(each setting gets a fresh batch, so cached launch geometry is recomputed).

    python tools/sweep_env.py "SMPM_GRID_MAX=8" "SMPM_GRID_MAX=32" ...
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1512_01756_b200 import Context  # noqa: E402
from paper_1512_01756_b200.configs import CONFIGS  # noqa: E402
from paper_1512_01756_b200.problems import build_problem, load_batch  # noqa: E402

cfg = CONFIGS[os.environ.get("SWEEP_CONFIG", "C4")]
ps = build_problem(cfg, device="cuda")
ctx = Context(0)
bS = torch.tensor(ps.b_S, device="cuda")
base = dict(os.environ)
for setting in [""] + sys.argv[1:]:
    os.environ.clear()
    os.environ.update(base)
    for kv in filter(None, setting.split(",")):
        k, v = kv.split("=")
        os.environ[k] = v
    b = load_batch(ctx, ps).tune_from_env()
    for _ in range(3):
        r = b.solve(bS, "dbj", 1e-10, 10 * cfg.max_iter, cfg.max_iter, "cgs2", True, history=False)
    torch.cuda.synchronize()
    ts = []
    for _ in range(7):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = b.solve(bS, "dbj", 1e-10, 10 * cfg.max_iter, cfg.max_iter, "cgs2", True, history=False)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    med = ts[len(ts) // 2]
    print(f"{setting or 'default':40s} median {med:.3f} ms  min {ts[0]:.3f}  solves/s {b.nsys / med * 1e3:.0f}  "
          f"iters max {max(r.iterations)} sum {sum(r.iterations)}", flush=True)
    b.close()
