"""Summarize SMPM_GT_TRACE dumps of the spectral grid tail: per-step phase times
(marks: 0 start, 1 T^-1 (first step), 2 per-mode pass, 4 T + coarse, 6 fused P,
7 CGS2 pass 1, 8 pass 2, 9 pass 3, 10 next-vector transform; 11 = live count)."""
import sys

import numpy as np

a = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(-1, 64, 16).astype(np.int64)
names = ["T^-1", "spec", "T+coarse", "-", "coarse read", "P", "pass1", "pass2", "pass3", "next-T^-1"]
for li, launch in enumerate(a):
    st = launch[(launch[:, 0] > 0) & (launch[:, 10] > 0)]
    if not len(st):
        continue
    d = np.diff(st[:, 1:11], axis=1) / 1e3
    d0 = (st[:, 1] - st[:, 0]) / 1e3
    live = st[:, 11]
    print(f"launch {li}: steps {len(st)} live {live.tolist()} mean step us {float((st[:, 10] - st[:, 0]).mean() / 1e3):.1f}")
    print("   mean us per phase:", {"T^-1": round(float(d0.mean()), 2),
                                    **{n: round(float(v), 2) for n, v in zip(names[1:], d.mean(axis=0))}})
    for Lv in sorted(set(live.tolist())):
        sel = live == Lv
        dd = d[sel].mean(axis=0)
        print(f"   L={Lv}: steps {int(sel.sum())} step us {float(((st[sel, 10] - st[sel, 0]) / 1e3).mean()):.1f}",
              {n: round(float(v), 2) for n, v in zip(names[1:], dd)})

