"""Median device time of warm solves of one config with a given method under SMPM_* settings.

    SWEEP_CONFIG=C3 python tools/sweep_method.py 2las "" "SMPM_GRID=0"
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1512_01756_b200 import Context  # noqa: E402
from paper_1512_01756_b200.configs import CONFIGS  # noqa: E402
from paper_1512_01756_b200.problems import build_problem, load_batch  # noqa: E402

cfg = CONFIGS[os.environ.get("SWEEP_CONFIG", "C3")]
method = sys.argv[1]
ps = build_problem(cfg, device="cuda")
ctx = Context(0)
bS = torch.tensor(ps.b_S, device="cuda")
base = dict(os.environ)
for setting in sys.argv[2:] or [""]:
    os.environ.clear()
    os.environ.update(base)
    for kv in filter(None, setting.split(",")):
        k, v = kv.split("=")
        os.environ[k] = v
    b = load_batch(ctx, ps).tune_from_env()
    for _ in range(2):
        r = b.solve(bS, method, 1e-10, 10 * cfg.max_iter, cfg.max_iter, "cgs2", True, history=False)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = b.solve(bS, method, 1e-10, 10 * cfg.max_iter, cfg.max_iter, "cgs2", True, history=False)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    print(f"{method} {setting or 'default':30s} median {ts[2]:.3f} ms  iters {sum(r.iterations)}", flush=True)
    b.close()
