"""Solve-only summary of an ncu launch list (`--metrics gpu__time_duration.sum --csv`) of
tools/prof_step.py: the launches before the solve's first kernel (zt_coarse_kernel) are the
device-side setup and are reported apart.

    python tools/launch_summary.py profiles/r02/launches_c5.csv.gz > profiles/r02/launches_c5_summary.txt
"""
import collections
import csv
import gzip
import re
import sys


def load(path):
    rows = list(csv.reader(gzip.open(path, "rt") if path.endswith(".gz") else open(path)))
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[start]
    col = {h: i for i, h in enumerate(hdr)}
    out = []
    for r in rows[start + 1:]:
        if len(r) == len(hdr) and r[col["Metric Name"]] == "gpu__time_duration.sum":
            name = re.sub(r"\(.*", "", r[col["Kernel Name"]])
            for junk in ("smpm::", "void ", "(anonymous namespace)::", "<unnamed>::"):
                name = name.replace(junk, "")
            v = float(r[col["Metric Value"]].replace(",", ""))
            out.append((name, v / 1e3 if r[col["Metric Unit"]] == "ns" else v))
    return out


seq = load(sys.argv[1])
i0 = next((i for i, (n, _) in enumerate(seq) if n.startswith("zt_coarse_kernel")), 0)
setup, solve = seq[:i0], seq[i0:]
tot = sum(v for _, v in solve)
print(f"{sys.argv[1]}: setup before the solve's first kernel: {len(setup)} launches, {sum(v for _, v in setup) / 1e3:.1f} ms")
print(f"one solve: {len(solve)} launches, {tot / 1e3:.1f} ms serialised (cold-cache per-launch times)")
agg = collections.OrderedDict()
for n, v in solve:
    a = agg.setdefault(n, [0, 0.0])
    a[0] += 1
    a[1] += v
for n, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"  {n[:46]:46s} n={c:4d} tot={v / 1e3:8.2f} ms  avg={v / c:8.1f} us  share {v / tot:6.1%}")
cls = collections.OrderedDict((k, 0.0) for k in ("transform", "orthogonalization", "per-mode pass", "other"))
for n, v in solve:
    k = ("transform" if n.startswith("xform") else "orthogonalization" if n.startswith("cgs")
         else "per-mode pass" if n.startswith("spec_op") else "other")
    cls[k] += v
print("classes:", ", ".join(f"{k} {v / tot:.1%}" for k, v in cls.items()))
