"""Summarize SMPM_GT_TRACE dumps: per-phase time of grid-persistent tail steps."""
import sys

import numpy as np

a = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(-1, 64, 16).astype(np.int64)
names = ["BJ1", "BJ2", "BJ3", "S", "Zt", "coarse+P", "pass1", "pass2", "pass3", "givens+scale"]
for li, launch in enumerate(a):
    st = launch[(launch[:, 0] > 0) & (launch[:, 10] > 0)]
    if not len(st):
        continue
    d = np.diff(st[:, :11], axis=1) / 1e3
    print(f"launch {li}: steps {len(st)} live {sorted(set(st[:, 11].tolist()))} "
          f"mean step us {float((st[:, 10] - st[:, 0]).mean() / 1e3):.1f}")
    print("   mean us per phase:", {n: round(float(v), 2) for n, v in zip(names, d.mean(axis=0))})
