"""Roofline of the operator kernels behind the C ABI (smpm_apply_S, smpm_apply_block_jacobi_inv)
at the BASELINE configs: device time per call with CUDA events on the launching stream (warm,
averaged over many calls, L2 flushed between calls), algorithmic flops and bytes per system from
DESIGN.md §4, fraction of the attainable roofline min(P_fp64, AI * B_HBM).

    python tools/op_roofline.py [--configs C2,C3,C4,C5] [--c5-modes 64] [--out file.json]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1512_01756_b200 import Context  # noqa: E402
import ctypes as C  # noqa: E402

from paper_1512_01756_b200._lib import lib  # noqa: E402
from paper_1512_01756_b200.configs import CONFIGS  # noqa: E402
from paper_1512_01756_b200.problems import build_problem, load_batch  # noqa: E402


def hbm_peak():
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6539.2, "fallback"


def counts(cfg):
    """Algorithmic flops / bytes per system per application."""
    w, d, mx, k = cfg.w, cfg.d, cfg.m_x, cfg.k
    nbf = d // 2
    odd = d % 2
    # S v = v + G_W v0 + G_E v_{2d-1} + G_I X (App. A): stored G_W, G_I, G_E once per system
    fS = 2 * ((2 * w) ** 2 * (mx - 2) + 2 * w * w) + k
    bS = 8 * ((2 * w) ** 2 + 2 * w * w + 2 * k)
    # structured block-Jacobi: per two-interface block 20 w^2 flops; stored G_I, G_W, G_E, the
    # K^-1 variants that occur (first / interior / last), K_single when d is odd; vectors v, tmp, y
    nvar = len({(bb == 0, 2 * bb + 2 == mx - 1) for bb in range(nbf)})
    fBJ = nbf * 20 * w * w + (6 * w * w if odd else 0)
    bBJ = 8 * (6 * w * w + nvar * 4 * w * w + (w * w if odd else 0) + 4 * k)
    return {"S": (fS, bS), "BJ": (fBJ, bBJ)}


def time_op(fn, v, reps, flush):
    st = torch.cuda.current_stream()
    for _ in range(3):
        fn(v)
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        fn(v)
        e1.record(st)
        e1.synchronize()
        tot += e0.elapsed_time(e1)
    return tot / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C2,C3,C4,C5")
    ap.add_argument("--c5-modes", type=int, default=64)
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    ctx = Context(0)
    df, dm = C.c_double(), C.c_double()
    lib().smpm_fp64_peak(0, C.byref(df), C.byref(dm))
    dfma, dmma = df.value, dm.value
    pf = max(dfma, dmma)
    bw, bw_src = hbm_peak()
    flush = torch.empty(256 * 2**20 // 8, dtype=torch.float64, device="cuda")  # > 126 MB L2
    rows = []
    for name in a.configs.split(","):
        cfg = CONFIGS[name]
        modes = None
        if name == "C5":
            modes = list(range(0, cfg.modes, max(1, cfg.modes // a.c5_modes)))[: a.c5_modes]
        ps = build_problem(cfg, modes=modes, device="cuda")
        b = load_batch(ctx, ps, spectral=False)
        ns = b.nsys
        v = torch.randn(ns, b.k, dtype=torch.float64, device="cuda")
        cnt = counts(cfg)
        for op, fn in (("S", b.apply_S), ("BJ", b.apply_block_jacobi_inv)):
            ms = time_op(fn, v, a.reps, flush)
            f, by = cnt[op]
            F, B = f * ns, by * ns
            ai = F / B
            att = min(pf * 1e12, ai * bw * 1e9)
            bound = "fp64" if pf * 1e12 <= ai * bw * 1e9 else "hbm"
            ach_f = F / (ms * 1e-3)
            row = {"config": name, "systems": ns, "op": op, "ms": ms, "gflop": F / 1e9, "mbytes": B / 1e6,
                   "ai": ai, "bound": bound, "tflops": ach_f / 1e12, "gbs": B / (ms * 1e-3) / 1e9,
                   "frac": ach_f / att}
            rows.append(row)
            print(json.dumps(row), flush=True)
        b.close()
        del ps
        torch.cuda.empty_cache()
    out = {"fp64_peak_tflops": pf, "dfma_tflops": dfma, "dmma_tflops": dmma, "hbm_gbs": bw, "hbm_source": bw_src,
           "rows": rows}
    if a.out:
        with open(a.out, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
