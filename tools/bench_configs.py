"""Solves/s of every BASELINE configuration on one GPU ("report GPU
solves/s at 1 GPU for all configs"), next to the oracle port of the reference on the
host cores (one thread, and all threads over independent systems).

GPU: device time of K warm batched solves (CUDA events on the launching stream,
inputs resident in HBM). CPU: the oracle port (reference per-interface layout, LU
block-Jacobi, Householder GMRES) on the product's couplings, a bounded sample.

    python tools/bench_configs.py [--configs C1,C2,C3,C4,C5] [--out profiles/r01/configs.json]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1512_01756_b200 import Context  # noqa: E402
from paper_1512_01756_b200.configs import CONFIGS  # noqa: E402
from paper_1512_01756_b200.problems import build_problem, load_batch  # noqa: E402


def gpu_rate(b, bS, method, sp, min_ms=300.0):
    def step():
        return b.solve(bS, method, sp["tol"], sp["max_iter"], sp["restart"], "cgs2", True, history=False)

    for _ in range(3 if min_ms > 0 else 1):
        r = step()
    torch.cuda.synchronize()
    k, ms = 1, 0.0
    while True:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(k):
            r = step()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        if ms >= min_ms or k >= 64:
            break
        k *= 2
    return b.nsys * k / (ms * 1e-3), ms / k, r, k


def run_c5(ctx, cfg, chunk):
    """C5 (256 modes, k = 277,440 each) in mode chunks (the Krylov basis of unrestarted
    GMRES up to 400 steps is 0.9 GB per mode), two regimes:
      * reference: GMRES with max_iter = 100 and no restart (the reference never
        restarts; BASELINE's GMRES(100)); modes that need more report not converged,
        exactly as the reference's KrylovReport would;
      * converged: unrestarted, max_iter = 400 (every mode converges; restarted
        GMRES(100) stagnates just above 1e-10 for the slow low modes)."""
    rows = []
    regimes = {"reference_max100": dict(tol=1e-10, max_iter=100, restart=0),
               "to_convergence": dict(tol=1e-10, max_iter=400, restart=0)}
    acc = {k: dict(ms=0.0, its=[], conv=[]) for k in regimes}
    setup_s = 0.0
    for c0 in range(0, cfg.modes, chunk):
        modes = list(range(c0, min(cfg.modes, c0 + chunk)))
        t0 = time.perf_counter()
        ps = build_problem(cfg, modes, device="cuda", device_rhs=True)
        b = load_batch(ctx, ps).tune_from_env()
        setup_s += time.perf_counter() - t0
        bS = torch.tensor(ps.b_S, device="cuda")
        for key, sp in regimes.items():
            _, ms, r, _ = gpu_rate(b, bS, "dbj", sp, min_ms=0.0)
            acc[key]["ms"] += ms
            acc[key]["its"] += list(r.iterations)
            acc[key]["conv"] += list(r.converged)
        b.close()
        del ps, bS, b
        torch.cuda.empty_cache()
    for key, sp in regimes.items():
        v = acc[key]
        row = {"config": cfg.name, "method": "dbj", "regime": key, **sp, "systems": cfg.modes,
               "k_per_system": cfg.k, "gpu_solves_per_s": cfg.modes / (v["ms"] * 1e-3),
               "gpu_ms_per_batch": v["ms"], "mode_chunk": chunk,
               "iterations_mean": float(np.mean(v["its"])), "iterations_max": int(max(v["its"])),
               "converged": bool(all(v["conv"])), "converged_modes": int(sum(v["conv"])),
               "setup_s_untimed": setup_s,
               "cpu_note": "not run: the reference layout needs 9.6 GB per C5 mode (2.47 TB for the batch); "
                           "see SURVEY.md §8(d)"}
        rows.append(row)
        print(json.dumps(row), flush=True)
    return rows


def run_3d(ctx, cfg):
    """The config as the 3D problem BASELINE describes ("3D Fourier-extended pressure
    solve", m_y = 2 x modes planes, L_y = cfg.l_y): transverse FFT -> schur_rhs ->
    batched independent dbj solves of all (mode, part) systems -> recovery -> inverse
    FFT, all on the device (paper_1512_01756_b200/solve3d.py); seeded smooth forcing."""
    from paper_1512_01756_b200.solve3d import Fourier3D

    m_y = 2 * cfg.modes
    t0 = time.perf_counter()
    solver = Fourier3D(ctx, cfg.n, cfg.m_x, cfg.m_z, cfg.l_x, cfg.l_z, m_y, cfg.l_y, cfg.c_tau)
    setup_s = time.perf_counter() - t0
    # every (mode, part) system carries the config's seeded per-mode forcing (real part:
    # stream j, imaginary part: stream modes + j; the j = 0 imaginary part of a real field
    # is zero): synthesize the coefficients and transform them back to the 3D field
    from paper_1512_01756_b200.problems import manufactured_batch
    from paper_1512_01756_b200.solve3d import inverse_fourier_y

    mus = solver.mus
    re = manufactured_batch(solver.geo, cfg.kmax, cfg.decay, cfg.seed, list(range(cfg.modes)), mus, "cuda")
    im = manufactured_batch(solver.geo, cfg.kmax, cfg.decay, cfg.seed, [cfg.modes + j for j in range(cfg.modes)],
                            mus, "cuda")
    im[0].zero_()
    coeff = torch.stack([re, im], dim=1).reshape(m_y, -1).contiguous()
    f = inverse_fourier_y(coeff, m_y)
    del re, im, coeff
    sp = bench.solve_params(cfg)
    for _ in range(2):
        res = solver.solve(f, "dbj", sp["tol"], sp["max_iter"], sp["restart"])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    nrep = 5
    e0.record()
    for _ in range(nrep):
        res = solver.solve(f, "dbj", sp["tol"], sp["max_iter"], sp["restart"])
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / nrep
    row = {"config": cfg.name + "-3D", "method": "dbj", "regime": "3D solve_3d on the device (FFT, rhs, solves, recovery, iFFT)",
           "m_y": m_y, "systems": 2 * cfg.modes, "nodes": int(f.shape[1]), "gpu_ms_per_3d_solve": ms,
           "gpu_3d_solves_per_s": 1e3 / ms, "gpu_system_solves_per_s": 2 * cfg.modes / (ms * 1e-3),
           "iterations_mean": float(np.mean(res.iterations)), "iterations_max": int(max(res.iterations)),
           "converged": bool(all(res.converged)), "stacked_rel_residual": res.rel_residual, "setup_s_untimed": setup_s,
           "forcing": "per-mode seeded cosine-mode fields (Lap - k_j^2) u_j as the C4 per-mode rhs, real part "
                      "stream j, imaginary part stream modes + j, synthesized through the inverse transform"}
    print(json.dumps(row), flush=True)
    return [row]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C1,C2,C3,C4,C5")
    ap.add_argument("--cpu-max-s", type=float, default=60.0, help="skip the CPU leg when one solve would exceed this")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--c5-chunk", type=int, default=64, help="C5 modes per batch")
    ap.add_argument("--no-stacked", action="store_true")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    ctx = Context(0)
    threads = os.cpu_count() or 1
    rows = []
    for name in a.configs.split(","):
        cfg = CONFIGS.get(name)
        if name == "C5":
            rows += run_c5(ctx, cfg, a.c5_chunk)
            continue
        if name.endswith("-3D"):
            rows += run_3d(ctx, CONFIGS[name[:-3]])
            continue
        sp = bench.solve_params(cfg)
        t0 = time.perf_counter()
        ps = build_problem(cfg, device="cuda")  # host FDM b_S, as bench.py
        b = load_batch(ctx, ps).tune_from_env()
        setup_s = time.perf_counter() - t0
        bS = torch.tensor(ps.b_S, device="cuda")
        for method in cfg.methods:
            rate, ms, r, k = gpu_rate(b, bS, method, sp)
            row = {"config": name, "method": method, "systems": b.nsys, "k_per_system": b.k,
                   "gpu_solves_per_s": rate, "gpu_ms_per_batch": ms, "timed_batches": k,
                   "iterations_mean": float(np.mean(r.iterations)), "iterations_max": int(max(r.iterations)),
                   "converged": bool(all(r.converged)), "setup_s_untimed": setup_s}
            # CPU legs: oracle port on the product couplings (bounded sample)
            if not a.no_cpu:
                idx = [ps.modes.index(m) for m in bench.sample_modes(cfg, threads)] if cfg.modes else [0]
                _, systems = bench.oracle_systems_from(ps, idx[:1], 1)
                dt1, its1 = bench.time_cpu(systems, ps.b_S[idx[:1]], 1, method, sp)
                row["cpu_1thread_solves_per_s"] = 1.0 / dt1
                row["cpu_1thread_sample"] = f"system {idx[0]} ({its1[0]} iterations)"
                if len(idx) > 1 and dt1 * len(idx) / threads < a.cpu_max_s:
                    _, systems = bench.oracle_systems_from(ps, idx, threads)
                    dtn, _ = bench.time_cpu(systems, ps.b_S[idx], threads, method, sp)
                    row["cpu_allcores_solves_per_s"] = len(idx) / dtn
                    row["cpu_allcores_sample"] = f"{len(idx)} systems, one per thread"
                elif not cfg.modes:
                    row["cpu_allcores_note"] = "one system: the reference has no intra-solve threading"
                row["cpu_threads"] = threads
            rows.append(row)
            print(json.dumps(row), flush=True)
        if cfg.modes and not a.no_stacked:
            # the reference bench's 3D default: one stacked GMRES over all modes
            # (proj/src/helmholtz.cpp:187-246, proj/src/bench.cpp:129), max_iter = 100, no restart
            def st():
                return b.solve_stacked(bS, "dbj", 1e-10, 100, 0, history=False)

            for _ in range(3):
                r = st()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            nrep = 5
            for _ in range(nrep):
                r = st()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / nrep
            row = {"config": name, "method": "dbj", "regime": "stacked (one GMRES over all modes)", "systems": b.nsys,
                   "k_per_system": b.k, "gpu_solves_per_s": b.nsys / (ms * 1e-3), "gpu_ms_per_batch": ms,
                   "iterations": int(r.iterations[0]), "converged": bool(r.converged[0]),
                   "final_rel_residual": float(r.final_rel_residual[0])}
            rows.append(row)
            print(json.dumps(row), flush=True)
        b.close()
        del ps, bS
        torch.cuda.empty_cache()
    out = {"cpu": bench.cpu_model(), "host_threads": threads, "rows": rows}
    if a.out:
        with open(a.out, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
