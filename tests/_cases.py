"""Test-case builders: oracle setups (the checker) for the BASELINE configs and
small grids, exported in the C-ABI's per-kind coupling layout."""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from oracle import oracle as O


@dataclass
class Case:
    prob: O.Problem
    systems: list            # oracle Systems (one per mode)
    mus: list
    b_S: np.ndarray          # nsys x k
    u_S: np.ndarray | None   # singular system's left null vector (mode 0)
    u_L: np.ndarray | None
    kinds: list = field(default_factory=list)  # (G_W, G_I, G_E) per system


def build_case(n, m_x, m_z, l_x, l_z, mus=(0.0,), kmax=4, decay=False, c_tau=2.0, seed=1234, streams=None,
               forcing_only=None, layout_reference=False, dense_limit=3200):
    prob = O.Problem(n, m_x, m_z, l_x, l_z, c_tau)
    systems, bs, kinds = [], [], []
    u_S = u_L = None
    streams = streams if streams is not None else list(range(len(mus)))
    for j, mu in enumerate(mus):
        s = O.System(prob, mu, layout_reference)
        s.build_bj()
        f, _ = prob.manufactured(kmax, decay, seed, streams[j], forcing_only=bool(forcing_only), mu=mu)
        if mu == 0.0:
            u_S, u_L, _, _ = s.nullspace(dense_limit)
            s.build_coarse(u_S)
            ft = O.project_out(f, u_L)
            b = O.project_out(s.schur_rhs(ft), u_S)
        else:
            s.build_coarse(None)
            b = prob.apply_B(prob.shifted_solve(mu, f))
        systems.append(s)
        bs.append(b)
        kinds.append(s.kinds())
    return Case(prob, systems, list(mus), np.array(bs), u_S, u_L, kinds)


def spectral_factors(case):
    """(npairs, T, T^-1, gamma) of the case's geometry and shifts (product FDM)."""
    from paper_1512_01756_b200.fdm import Geometry, StripFDM

    p = case.prob
    geo = Geometry(p.n, p.m_x, p.m_z, p.l_x, p.l_z, p.c_tau)
    return StripFDM(geo, device="cpu").spectral(case.mus)


def gpu_batch(ctx, case, prob_dims=None, spectral=False):
    """SchurBatch with the oracle's dense couplings (the reference data); with
    spectral=True also the product's spectral factors of the same geometry."""
    from paper_1512_01756_b200 import SchurBatch

    p = case.prob
    b = SchurBatch(ctx, p.n, p.m_x, p.m_z, len(case.systems))
    for i, (gw, gi, ge) in enumerate(case.kinds):
        b.set_couplings(i, gw, gi if p.m_x > 2 else None, ge)
        if case.mus[i] == 0.0:
            b.set_nullspace(i, case.u_S)
    if spectral:
        b.set_spectral(*spectral_factors(case))
    return b.finalize()


def rel(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
