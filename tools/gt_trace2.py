"""Summarize SMPM_GT_TRACE2 dumps: per-CTA timing inside the grid tail's operator stages
(last launch in the file; times relative to the earliest stage start)."""
import sys

import numpy as np

raw = np.fromfile(sys.argv[1], dtype=np.uint64).astype(np.int64)
pos, launches = 0, []
while pos < len(raw):
    nb = int(raw[pos]); pos += 1
    launches.append(raw[pos:pos + 16 * nb * 8].reshape(4, 4, nb, 8)); pos += 16 * nb * 8
a = launches[int(sys.argv[2]) if len(sys.argv) > 2 else -1]
names = ["BJ1", "BJ2", "BJ3", "S"]


def q(v):
    return f"{np.median(v)/1e3:.2f}/{v.max()/1e3:.2f}" if len(v) else "-"


for step in range(4):
    for stg in range(4):
        x = a[step, stg]
        ok = x[:, 0] > 0
        if not ok.any():
            continue
        t0 = x[ok, 0].min()
        g = x[:, 1] > 0
        v = x[:, 5] > 0
        print(f"step {step} {names[stg]}: start {q(x[ok,0]-t0)} | gemm ctas {g.sum()}: mainloop end {q(x[g,1]-t0)} "
              f"reduce end {q(x[g,2]-t0)} clsync end {q(x[g,3]-t0)} | gemv ctas {v.sum()}: start {q(x[v,4]-t0)} end {q(x[v,5]-t0)}")
