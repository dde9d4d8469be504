"""Summarize SMPM_CL_TRACE dumps: per-phase time of cluster Arnoldi steps."""
import sys

import numpy as np

a = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(-1, 64, 12).astype(np.int64)
names = ["BJ1", "BJ2", "BJ3", "S", "P", "pass1", "pass2", "pass3", "givens+scale"]
steps = a[(a[:, :, 0] > 0) & (a[:, :, 9] > 0)]
print("steps traced", len(steps))
d = np.diff(steps[:, :10], axis=1) / 1e3
print("mean us per phase:", {n: round(float(v), 1) for n, v in zip(names, d.mean(axis=0))})
print("mean step us", round(float((steps[:, 9] - steps[:, 0]).mean() / 1e3), 1))
t0 = a[a > 0].min() if (a > 0).any() else 0
span = (a[:, :, 9].max() - a[:, :, 0][a[:, :, 0] > 0].min()) / 1e3
print("kernel span us (traced)", round(float(span), 1))
