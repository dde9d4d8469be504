"""profiles/rNN/traffic.json from ncu --set full raw-page CSVs (exported on the GPU
box with `ncu -i X.ncu-rep --page raw --csv`): DRAM bytes (dram__bytes_read.sum +
dram__bytes_write.sum) and duration of the launch group of each kernel class at a
stated point (live systems, Arnoldi index j), next to the algorithmic bytes of the
SAME launch group (SURVEY §8(d) and the implementation minimum, as
bench.algorithmic_counts), so traffic / algorithmic is a wasted-traffic ratio.

    python tools/make_traffic.py --config C5 --out profiles/r02/traffic.json \
        --cgs profiles/r02/cgs_j40_12sys.csv.gz --cgs-live 10 --cgs-j 40 \
        --xform profiles/r02/xform_spec_64sys.csv.gz --xform-live 64
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1512_01756_b200.configs import CONFIGS  # noqa: E402
from tools.ncu_traffic import launches  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    ap.add_argument("--cgs")
    ap.add_argument("--cgs-live", type=int)
    ap.add_argument("--cgs-j", type=int)
    ap.add_argument("--xform")
    ap.add_argument("--xform-live", type=int)
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    k, w, d = cfg.k, cfg.w, cfg.m_x - 1
    res = {"config": cfg.name, "note": "ncu --set full, --clock-control none, cold per-launch replay; bytes per "
           "launch group at the stated point", "classes": {}}
    if a.cgs:
        ls = [x for x in launches(a.cgs) if "cgs" in x["kernel"]][:2]
        live, j = a.cgs_live, a.cgs_j
        dram = sum(x["dram_bytes"] for x in ls)
        t = sum(x["duration_s"] for x in ls)
        s8d = live * 8.0 * k * (j + 2)
        impl = live * 8.0 * k * (2 * (j + 1) + 5)
        res["classes"]["orthogonalization"] = {
            "kernels": [x["kernel"] for x in ls], "live": live, "j": j, "dram_bytes": dram,
            "s8d_bytes": s8d, "impl_min_bytes": impl, "traffic_over_impl_min": dram / impl,
            "traffic_over_s8d": dram / s8d, "duration_s": t, "dram_gbs": dram / t / 1e9,
            "per_kernel": [{"kernel": x["kernel"], "grid": x["grid"], "dram_bytes": x["dram_bytes"],
                            "duration_s": x["duration_s"], "dram_gbs": x["dram_bytes"] / x["duration_s"] / 1e9}
                           for x in ls],
            "note": "deferred CGS2: pass 1B (j old columns + the pending pair) and pass 2' (j + 1 columns)"}
    if a.xform:
        ls = launches(a.xform)
        live = a.xform_live
        xf = [x for x in ls if "xformp" in x["kernel"] or "xformq" in x["kernel"]][:2]
        spo = [x for x in ls if "spec_op" in x["kernel"]][:1]
        vec = live * 2.0 * k * 8
        res["classes"]["transform"] = {
            "live": live, "dram_bytes": sum(x["dram_bytes"] for x in xf),
            "impl_min_bytes": 2 * vec, "s8d_bytes": 2 * vec,
            "traffic_over_impl_min": sum(x["dram_bytes"] for x in xf) / (2 * vec),
            "duration_s": sum(x["duration_s"] for x in xf),
            "flops_per_launch": live * 2.0 * d * w * w,
            "per_kernel": [{"kernel": x["kernel"], "grid": x["grid"], "dram_bytes": x["dram_bytes"],
                            "duration_s": x["duration_s"],
                            "tflops": live * 2.0 * d * w * w / x["duration_s"] / 1e12} for x in xf],
            "note": "parity-split T^-1 and T of one Arnoldi step: 2 d columns per system, w x (w/2) x 2 flops "
                    "per column and direction; the vectors (one read, one write of k doubles per system and "
                    "direction) are the algorithmic traffic, the shared matrix streams from L2"}
        if spo:
            x = spo[0]
            res["classes"]["spectral_op"] = {
                "live": live, "kernels": [x["kernel"]], "dram_bytes": x["dram_bytes"], "impl_min_bytes": vec,
                "s8d_bytes": vec, "traffic_over_impl_min": x["dram_bytes"] / vec, "duration_s": x["duration_s"],
                "dram_gbs": x["dram_bytes"] / x["duration_s"] / 1e9}
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
