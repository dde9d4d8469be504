"""GPU timeline of one warm batched solve via torch.profiler (CUPTI): every
kernel / memcpy with start, duration and the idle gap before it."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_1512_01756_b200 import Context  # noqa: E402
from paper_1512_01756_b200.configs import CONFIGS  # noqa: E402
from paper_1512_01756_b200.problems import build_problem, load_batch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--rows", type=int, default=400)
a = ap.parse_args()
cfg = CONFIGS[a.config]
ps = build_problem(cfg, device="cuda")
ctx = Context(0)
b = load_batch(ctx, ps).tune_from_env()
bS = torch.tensor(ps.b_S, device="cuda")
for _ in range(2):
    b.solve(bS, "dbj", 1e-10, 10 * cfg.max_iter, cfg.max_iter, "cgs2", True, history=False)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    b.solve(bS, "dbj", 1e-10, 10 * cfg.max_iter, cfg.max_iter, "cgs2", True, history=False)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
ev.sort(key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
busy = 0.0
prev_end = t0
rows = []
for e in ev:
    st, en = e.time_range.start, e.time_range.end
    gap = st - prev_end
    busy += en - st
    rows.append((st - t0, en - st, gap, e.name))
    prev_end = max(prev_end, en)
span = prev_end - t0
print(f"events {len(ev)}  span {span:.1f} us  busy {busy:.1f} us  idle {span - busy:.1f} us")
agg = {}
for _, du, gap, name in rows:
    k = name.split("(")[0].split("<")[0].split("::")[-1][:40]
    a_ = agg.setdefault(k, [0, 0.0, 0.0])
    a_[0] += 1
    a_[1] += du
    a_[2] += max(gap, 0)
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"  {k:40s} n={v[0]:4d} busy={v[1]:8.1f}us gaps-before={v[2]:8.1f}us")
for st, du, gap, name in rows[: a.rows]:
    print(f"{st:9.1f} {du:8.1f} gap {gap:7.1f}  {name[:70]}")
