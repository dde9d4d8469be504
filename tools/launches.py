"""Summarize an ncu launch-list CSV (gpu__time_duration.sum) for the last solve."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
idx = [i for i, d in enumerate(data) if "gm_start" in d["Kernel Name"]]
last = data[idx[-1] - 4:]
agg = collections.OrderedDict()
for d in last:
    name = d["Kernel Name"].split("(")[0].split("::")[-1]
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += float(d["Metric Value"])
tot = sum(a[1] for a in agg.values())
print(f"launches {len(last)}  total {tot/1e3:.1f} us")
for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"  {k[:34]:34s} n={a[0]:4d} tot={a[1]/1e3:8.1f}us avg={a[1]/a[0]/1e3:6.1f}us")
if len(sys.argv) > 2:
    line = [f"{d['Kernel Name'].split('(')[0].split('::')[-1][:9]}:{float(d['Metric Value'])/1e3:.0f}" for d in last]
    n = int(sys.argv[2])
    for i in range(0, min(n, len(line)), 12):
        print("   " + " ".join(line[i:i + 12]))
    print("   ...")
    for i in range(max(0, len(line) - n), len(line), 12):
        print("   " + " ".join(line[i:i + 12]))
