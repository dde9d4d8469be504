"""profiles/rNN/traffic.json from ncu --set full reports of the bench workload:
DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) of one launch group of
a kernel class at a stated point (live systems, Arnoldi index j), next to the
algorithmic bytes of the SAME launch group (SURVEY §8(d) and the implementation
minimum, bench.algorithmic_counts' per-step terms), so traffic / algorithmic is
a wasted-traffic ratio.

    python tools/ncu_traffic.py --config C5 --cgs3 cgs3_fullbatch.ncu-rep \
        [--xform xformk.ncu-rep] [--spec spec_op.ncu-rep] --out profiles/r02/traffic.json
"""
import argparse
import csv
import io
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1512_01756_b200.configs import CONFIGS  # noqa: E402

SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def launches(path):
    if path.endswith((".csv", ".csv.gz")):  # raw page exported on the GPU box
        import gzip

        raw = (gzip.open if path.endswith(".gz") else open)(path, "rt").read()
    else:
        raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    out = []
    for r in data:
        def num(name):
            v = r[col[name]].replace(",", "")
            return float(v) * SCALE.get(units[col[name]], 1.0)

        dur = float(r[col["gpu__time_duration.sum"]].replace(",", ""))
        dscale = {"nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "second": 1.0, "s": 1.0}.get(units[col["gpu__time_duration.sum"]], 1e-9)
        out.append({"kernel": r[col["Kernel Name"]].split("(")[0].replace("smpm::", ""), "grid": r[col["Grid Size"]],
                    "dram_bytes": num("dram__bytes_read.sum") + num("dram__bytes_write.sum"),
                    "duration_s": dur * dscale})
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    ap.add_argument("--cgs3", help="report of the first full-batch step's three CGS2 passes (j = 0)")
    ap.add_argument("--live", type=int, default=0, help="live systems of that step (default: all)")
    ap.add_argument("--xform", help="report of full-batch transform launches")
    ap.add_argument("--spec", help="report of full-batch per-mode passes")
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    k, w, d = cfg.k, cfg.w, cfg.m_x - 1
    live = a.live or max(cfg.modes, 1)
    res = {"config": cfg.name, "note": "ncu --set full, --clock-control none, cold per-launch replay", "classes": {}}
    if a.cgs3:
        ls = launches(a.cgs3)[:3]
        j = 0
        dram = sum(x["dram_bytes"] for x in ls)
        s8d = live * 8.0 * k * (j + 2)
        impl = live * 8.0 * k * (3 * (j + 1) + 7)
        t = sum(x["duration_s"] for x in ls)
        res["classes"]["orthogonalization"] = {
            "kernels": [x["kernel"] for x in ls], "live": live, "j": j, "dram_bytes": dram,
            "s8d_bytes": s8d, "impl_min_bytes": impl, "traffic_over_impl_min": dram / impl,
            "traffic_over_s8d": dram / s8d, "duration_s": t, "dram_gbs": dram / t / 1e9}
    if a.xform:
        ls = launches(a.xform)
        res["classes"]["transform"] = {"launches": ls, "note": "DRAM bytes of each launch; the algorithmic vector "
                                       "traffic of one full-batch transform is 2 k doubles per system"}
    if a.spec:
        ls = launches(a.spec)
        res["classes"]["spectral_op"] = {"launches": ls, "algorithmic_bytes_per_launch": live * 2.0 * k * 8}
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
