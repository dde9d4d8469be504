"""Parity of the product path (load_batch: product couplings + spectral operator,
the path bench.py times) against the oracle on identical inputs, at the BASELINE
configurations, with the oracle's OWN input sensitivity as the envelope.

Why an envelope.  Many Fourier modes converge fast to ~1e-9 and then plateau
within a factor 2-5 of the 1e-10 target, where the GMRES residual
estimate moves with rounding.  On such a mode two valid implementations (or the
same implementation on inputs that differ in the 13th digit) stop at different
iterations.  So every comparison here runs the oracle on the right-hand side and
on copies perturbed by 1e-13 relative (seeded), and holds the GPU to:
  * iterations exactly +-1 of the unperturbed oracle wherever the oracle itself
    is stable (its perturbed runs agree with it within +-1); on an unstable
    (plateau) mode, a stop inside the plateau: no earlier than the first step at
    which the oracle's own residual history comes within PLATEAU_F = 5 of the
    target (these modes plateau within a factor 2-5 of it) and no
    later than the slowest perturbed oracle run (+1).  Measured on C5 modes 3
    and 8: the oracle stops at 86 / 81 on b_S and at 226-236 on 1e-13
    perturbations of it, the GPU at 69 / 48;
  * residual histories entrywise (1e-10 + 1e-6 h) while h >= 1e-6, decade
    crossings +-1 on stable modes;
  * x_S within 1e-10 relative of the oracle (mean-removed for the singular
    mode 0), or, where the oracle's perturbed runs themselves move x_S by more,
    within 2x the oracle's own spread.
GMRES(m) is run as the reference runs it: one Krylov space of at most m
vectors, no restart (proj/src/gmres.cpp:35), plus the unrestarted-to-convergence
regime where GMRES(100) stops short (C5).  References: deflated_solve
proj/src/deflation.cpp:102-122, two_level_schwarz_solve :124-143, gmres
proj/src/gmres.cpp:18-142.

SMPM_PARITY_OUT=<dir>: each test also writes its per-mode table there (JSON).
"""
import json
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from oracle import oracle as O
from paper_1512_01756_b200 import configs
from paper_1512_01756_b200.problems import build_problem, load_batch
from tests.test_gpu_configs import _hist_ok

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

SOL_TOL = 1e-10
PERTURB = 1e-13
PLATEAU_F = 5.0
THREADS = max(1, os.cpu_count() or 1)


def _rel(x, ref, singular):
    if singular:  # x_S is defined up to the constant null direction (SURVEY convention 7)
        x, ref = x - x.mean(), ref - ref.mean()
    return float(np.linalg.norm(x - ref) / max(np.linalg.norm(ref), 1e-300))


def perturbed(b, seed):
    """b with every entry scaled by (1 + 1e-13 xi), xi ~ N(0, 1) (seeded)."""
    xi = np.random.default_rng(1000 + seed).standard_normal(b.shape)
    return b * (1.0 + PERTURB * xi)


def oracle_systems(ps, layout_reference=False):
    """Oracle systems on the product's couplings (the oracle's dedup layout: one
    stored coupling per strip kind, shared LU per distinct block-Jacobi block;
    bitwise the same entries as the reference layout, proj/src/schur.cpp:113-124)."""
    cfg = ps.cfg
    O.set_threads(1)
    prob = O.Problem(cfg.n, cfg.m_x, cfg.m_z, cfg.l_x, cfg.l_z, cfg.c_tau)

    def make(i):
        s = O.System(prob, ps.mus[i], layout_reference, kinds=(ps.GW[i], ps.GI[i] if cfg.m_x > 2 else None, ps.GE[i]))
        s.build_bj(1)
        s.build_coarse(ps.u_S if ps.mus[i] == 0.0 else None)
        return s

    with ThreadPoolExecutor(THREADS) as ex:
        systems = list(ex.map(make, range(len(ps.mus))))
    return prob, systems


def run_jobs(jobs):
    """jobs: list of (system, b, method, tol, max_iter) -> oracle SolveResults,
    solved concurrently (ctypes releases the GIL; the solve path is read-only)."""
    def one(j):
        s, b, method, tol, mi = j
        return s.solve(b, method, tol, mi, 0)

    with ThreadPoolExecutor(min(THREADS, len(jobs))) as ex:
        return list(ex.map(one, jobs))


def compare_modes(res, ps, base, perts, labels=None, resolved=1e-6, systems=None, method="dbj", tol=1e-10):
    """Per-mode parity of a GPU solve `res` against the oracle base runs and
    their perturbed re-runs (perts[i]: list of SolveResults for system i).
    Returns (rows, failures): the per-mode table and the bars of the module
    docstring each row misses (asserted by the caller after the table is dumped).
    `systems` (the oracle systems) gives the plateau entry of unstable modes."""
    rows, fails = [], []
    x = res.x_S.cpu().numpy()
    for i in range(len(base)):
        sing = ps.mus[i] == 0.0
        ref = base[i]
        its_all = [ref.iterations] + [p.iterations for p in perts[i]]
        lo, hi = min(its_all), max(its_all)
        stable = hi - lo <= 1
        spread = max([_rel(p.x_S, ref.x_S, sing) for p in perts[i]] + [0.0])
        err = _rel(x[i], ref.x_S, sing)
        g = int(res.iterations[i])
        row = {"system": labels[i] if labels else i, "mu": ps.mus[i], "gpu_iterations": g,
               "oracle_iterations": ref.iterations, "oracle_perturbed_iterations": its_all[1:],
               "oracle_stable": stable, "x_rel_err": err, "oracle_x_spread": spread,
               "gpu_converged": bool(res.converged[i]), "oracle_converged": bool(ref.converged),
               "oracle_perturbed_converged": [bool(p.converged) for p in perts[i]],
               "gpu_final_rel": float(res.final_rel_residual[i]), "oracle_final_rel": ref.final_rel_residual}
        bad = []
        if stable:
            if abs(g - ref.iterations) > 1:
                bad.append("iterations not +-1 on a stable mode")
        else:
            entry = lo
            if systems is not None:
                b = ps.b_S[i]
                rhs = systems[i].apply_P(b) if method == "dbj" else b
                target_h = tol * np.linalg.norm(b) / np.linalg.norm(rhs)
                near = np.nonzero(ref.history <= PLATEAU_F * target_h)[0]
                entry = int(near[0]) if near.size else lo
                row["plateau_entry"] = entry
                row["target_in_history_units"] = float(target_h)
                row["oracle_history_tail"] = [float(v) for v in ref.history[max(0, entry - 2):ref.iterations + 1]]
                if res.histories:
                    row["gpu_history_tail"] = [float(v) for v in res.histories[i][max(0, entry - 2):g + 1]]
            if not entry - 1 <= g <= hi + 1:
                bad.append("stop outside the plateau window [oracle plateau entry, slowest oracle run]")
        if err > max(SOL_TOL, 2.0 * spread):
            bad.append("x_S beyond max(1e-10, 2x the oracle's own spread)")
        if res.histories:
            try:
                if stable:
                    _hist_ok(res.histories[i], ref.history, resolved=resolved)
                else:
                    _hist_entrywise(res.histories[i], ref.history, resolved)
            except AssertionError:
                bad.append("history")
        row["failed"] = bad
        rows.append(row)
        if bad:
            fails.append((row["system"], bad))
    return rows, fails


def _hist_entrywise(h, ref, resolved=1e-6):
    n = min(len(h), len(ref))
    hi = ref[:n] >= resolved
    assert np.all(np.abs(h[:n] - ref[:n])[hi] <= 1e-10 + 1e-6 * ref[:n][hi])


def _dump(name, payload):
    out = os.environ.get("SMPM_PARITY_OUT")
    if out:
        os.makedirs(out, exist_ok=True)
        with open(os.path.join(out, name + ".json"), "w") as f:
            json.dump(payload, f, indent=1, default=float)


def _summary(rows):
    g = np.array([r["gpu_iterations"] for r in rows])
    o = np.array([r["oracle_iterations"] for r in rows])
    st = np.array([r["oracle_stable"] for r in rows])
    return {"systems": len(rows), "gpu_iterations_total": int(g.sum()), "oracle_iterations_total": int(o.sum()),
            "within_1_of_oracle": int((np.abs(g - o) <= 1).sum()), "oracle_stable_systems": int(st.sum()),
            "oracle_perturbed_totals": [int(sum(r["oracle_perturbed_iterations"][k] for r in rows))
                                        for k in range(len(rows[0]["oracle_perturbed_iterations"]))],
            "max_x_rel_err_stable": float(max([r["x_rel_err"] for r in rows if r["oracle_stable"]] + [0.0]))}


def test_c4_all_modes(ctx):
    """All 128 C4 modes through the product path vs the oracle on the same
    couplings and b_S, GMRES(100), with two 1e-13-perturbed oracle re-runs."""
    import torch

    cfg = configs.C4
    ps = build_problem(cfg, device="cuda")
    b = load_batch(ctx, ps)
    res = b.solve(torch.tensor(ps.b_S, device="cuda"), "dbj", 1e-10, cfg.max_iter, 0)
    _, systems = oracle_systems(ps)
    nsys = len(systems)
    rhs = [ps.b_S, perturbed(ps.b_S, 1), perturbed(ps.b_S, 2)]
    jobs = [(systems[i], r[i], "dbj", 1e-10, cfg.max_iter) for r in rhs for i in range(nsys)]
    out = run_jobs(jobs)
    base = out[:nsys]
    perts = [[out[nsys + i], out[2 * nsys + i]] for i in range(nsys)]
    rows, fails = compare_modes(res, ps, base, perts, labels=ps.modes, systems=systems)
    summ = _summary(rows)
    _dump("parity_c4_all_modes", {"config": "C4", "gmres": "max_iter 100, no restart", "summary": summ, "modes": rows})
    print(json.dumps(summ))
    assert not fails, fails
    assert summ["within_1_of_oracle"] >= summ["oracle_stable_systems"]


@pytest.mark.parametrize("name", ["C2", "C3"])
def test_2d_product_path(ctx, name):
    """C2 / C3 through the product path (spectral operator, load_batch default),
    dbj (and 2LAS at C3), GMRES(50/100) as the reference runs it."""
    import torch

    cfg = configs.CONFIGS[name]
    ps = build_problem(cfg, device="cuda")
    b = load_batch(ctx, ps)
    assert b.spectral
    _, systems = oracle_systems(ps)
    payload = {"config": name}
    fails = []
    for method in cfg.methods:
        res = b.solve(torch.tensor(ps.b_S, device="cuda"), method, 1e-10, cfg.max_iter, 0)
        rhs = [ps.b_S] + [perturbed(ps.b_S, q) for q in (1, 2, 3)]
        out = run_jobs([(systems[0], r[0], method, 1e-10, cfg.max_iter) for r in rhs])
        # 2LAS at C3 stagnates near 1e-6 for a stretch, where the residual estimates of
        # two valid implementations differ by ~1 %: entrywise histories while h >= 1e-4
        rows, f = compare_modes(res, ps, [out[0]], [out[1:]], resolved=1e-4 if method == "2las" else 1e-6,
                                systems=systems, method=method)
        payload[method] = rows[0]
        fails += [(method, x) for x in f]
        print(name, method, json.dumps(rows[0]))
    _dump(f"parity_{name.lower()}_product", payload)
    assert not fails, fails


def test_c5_modes(ctx):
    """C5 (k = 277,440) modes 0, 3, 8, 255 through the product path (device b_S,
    as bench.py), under GMRES(100) (the reference's max_iter = 100: modes 3 and 8
    stop short of 1e-10, converged = false on both sides) and unrestarted to
    convergence (max_iter 300), each against the oracle and a 1e-13-perturbed
    oracle re-run on the same couplings and b_S."""
    import torch

    cfg = configs.C5
    modes = [0, 3, 8, 255]
    ps = build_problem(cfg, modes, device="cuda", device_rhs=True)
    b = load_batch(ctx, ps)
    bS = torch.tensor(ps.b_S, device="cuda")
    _, systems = oracle_systems(ps)
    n = len(modes)
    pert = [perturbed(ps.b_S, q) for q in (1, 2, 3)]
    regimes = {"gmres100": 100, "unrestarted": 300}
    jobs, keys = [], []
    for reg, mi in regimes.items():
        for i in range(n):
            for tag, rhs in [("base", ps.b_S)] + [(f"p{q}", p) for q, p in enumerate(pert)]:
                jobs.append((systems[i], rhs[i], "dbj", 1e-10, mi))
                keys.append((reg, i, tag))
    out = dict(zip(keys, run_jobs(jobs)))
    payload = {"config": "C5", "modes": modes, "b_S": "device strip solves (schur_rhs), as bench.py",
               "perturbation": "b_S * (1 + 1e-13 xi), xi ~ N(0,1), seeds 1..3"}
    fails = []
    for reg, mi in regimes.items():
        res = b.solve(bS, "dbj", 1e-10, mi, 0)
        base = [out[(reg, i, "base")] for i in range(n)]
        perts = [[out[(reg, i, f"p{q}")] for q in range(3)] for i in range(n)]
        rows, f = compare_modes(res, ps, base, perts, labels=modes, systems=systems)
        payload[reg] = rows
        fails += [(reg, x) for x in f]
        for r in rows:
            print(reg, json.dumps(r))
    _dump("parity_c5_modes", payload)
    assert not fails, fails
