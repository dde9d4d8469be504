"""CPU tests of the product's host side: seeded inputs, the FDM setup against
the oracle's LU / real-Schur setup, configs, and the C-ABI export table."""
import ctypes
import os
import re

import numpy as np
import pytest

from oracle import oracle as O
from paper_1512_01756_b200 import configs, fdm, problems
from paper_1512_01756_b200._lib import EXPORTS, LIB_PATH

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_rng_bit_exact_with_cpp_engine():
    g = np.load(os.path.join(GOLD, "rng.npz"))
    for t in range(4):
        r = problems.Rng(1234).stream(t)
        mine = np.array([r.uniform() for _ in range(8)])
        assert np.array_equal(mine, g[f"uniform_{t}"])
        assert np.array_equal(mine, O.rng_uniforms(1234, t, 8))
    r = problems.Rng(0x5EED0001)
    assert np.array_equal(np.array([r.uniform() - 0.5 for _ in range(8)]), g["nullspace_start"])


@pytest.mark.parametrize("mu", [0.0, 3.0])
def test_manufactured_matches_oracle(mu):
    geo = fdm.Geometry(9, 4, 4, 1.0, 1.0)
    p = O.Problem(9, 4, 4, 1.0, 1.0, 2.0)
    f1, u1 = problems.manufactured(geo, 4, False, 1234, 2, mu=mu)
    f2, u2 = p.manufactured(4, False, 1234, 2, mu=mu)
    assert np.abs(f1 - f2).max() <= 1e-12 * np.abs(f2).max()
    assert np.abs(u1 - u2).max() <= 1e-13


def test_gll_product_matches_oracle():
    for n in (2, 3, 5, 9, 13, 17):
        x1, w1, d1 = fdm.gll_nodes(n)
        x2, w2, d2 = O.gll(n)
        assert np.allclose(x1, x2, rtol=0, atol=2e-16) and np.allclose(w1, w2, rtol=1e-14, atol=0) and np.allclose(d1, d2, rtol=0, atol=1e-13 * np.abs(d2).max())


GRIDS = [(9, 4, 4, 1.0, 1.0, 0.0), (6, 6, 4, 24.0, 4.0, 0.0), (6, 2, 3, 2.0, 1.0, 0.0), (7, 5, 3, 5.0, 1.0, 2.5),
         (11, 6, 16, 16.0, 1.0, (2 * np.pi * 5 / 16) ** 2)]


@pytest.mark.parametrize("grid", GRIDS)
def test_fdm_couplings_match_oracle(grid):
    """Kronecker-sum fast diagonalization vs the reference's LU / real-Schur couplings."""
    n, mx, mz, lx, lz, mu = grid
    p = O.Problem(n, mx, mz, lx, lz, 2.0)
    s = O.System(p, mu, False)
    gw, gi, ge = s.kinds()
    F = fdm.StripFDM(fdm.Geometry(n, mx, mz, lx, lz), "cpu")
    GW, GI, GE = F.couplings([mu])
    tol = 1e-10
    assert np.abs(GW[0] - gw).max() <= tol * np.abs(gw).max()
    assert np.abs(GE[0] - ge).max() <= tol * np.abs(ge).max()
    if mx > 2:
        assert np.abs(GI[0] - gi).max() <= tol * np.abs(gi).max()
    assert F.max_imag <= 1e-10 * max(np.abs(gw).max(), 1.0)
    f, _ = p.manufactured(4, True, 1234, 0, mu=mu)
    ref = s.schur_rhs(f) if mu == 0.0 else p.apply_B(p.shifted_solve(mu, f))
    assert np.linalg.norm(F.schur_rhs(f, mu) - ref) <= 1e-8 * np.linalg.norm(ref)


def _pair_block_apply(npairs, T, Ti, gam):
    """Dense T diag(gamma) T^-1 of the spectral form (pairs act on z = a - i b)."""
    w = T.shape[0]
    D = np.zeros((w, w))
    for t in range(npairs):
        g = gam[t]
        D[2 * t:2 * t + 2, 2 * t:2 * t + 2] = [[g.real, g.imag], [-g.imag, g.real]]
    for t in range(npairs, len(gam)):
        D[npairs + t, npairs + t] = gam[t].real
    return T @ D @ Ti


@pytest.mark.parametrize("grid", GRIDS)
def test_spectral_factors_reproduce_oracle_couplings(grid):
    """smpm_batch_set_spectral data: T diag(gamma_kind) T^-1 equals the
    reference's dense couplings G_W, G_I (four blocks), G_E."""
    n, mx, mz, lx, lz, mu = grid
    p = O.Problem(n, mx, mz, lx, lz, 2.0)
    gw, gi, ge = O.System(p, mu, False).kinds()
    F = fdm.StripFDM(fdm.Geometry(n, mx, mz, lx, lz), "cpu")
    npairs, T, Ti, gam = F.spectral([mu])
    w = T.shape[0]
    assert gam.shape == (1, 6, w - npairs)
    assert np.abs(T @ Ti - np.eye(w)).max() < 1e-10
    blocks = {0: gw, 5: ge}
    if mx > 2:
        blocks.update({1: gi[:w, :w], 2: gi[:w, w:], 3: gi[w:, :w], 4: gi[w:, w:]})
    for kind, ref in blocks.items():
        G = _pair_block_apply(npairs, T, Ti, gam[0, kind])
        assert np.abs(G - ref).max() <= 1e-10 * np.abs(ref).max(), kind


@pytest.mark.parametrize("grid", [g for g in GRIDS if g[5] == 0.0])
def test_fdm_null_vectors_match_oracle(grid):
    n, mx, mz, lx, lz, _ = grid
    p = O.Problem(n, mx, mz, lx, lz, 2.0)
    s = O.System(p, 0.0, False)
    uS, uL, _, _ = s.nullspace()
    F = fdm.StripFDM(fdm.Geometry(n, mx, mz, lx, lz), "cpu")
    fS, fL = F.nullspace()
    assert np.abs(fS - uS).max() <= 1e-9 and np.abs(fL - uL).max() <= 1e-9


def test_problem_builder_c1_matches_oracle():
    ps = problems.build_problem(configs.C1, device="cpu")
    g = np.load(os.path.join(GOLD, "c1_dbj.npz"))
    assert np.linalg.norm(ps.b_S[0] - g["b_S"]) <= 1e-9 * np.linalg.norm(g["b_S"])


def test_config_sizes():
    # SURVEY.md §8(a) table
    sizes = {c: (cfg.w, cfg.k, cfg.d) for c, cfg in configs.CONFIGS.items()}
    assert sizes == {"C1": (36, 216, 3), "C2": (416, 25792, 31), "C3": (272, 69088, 127),
                     "C4": (176, 22176, 63), "C5": (544, 277440, 255)}
    assert len(configs.C4.mus()) == 128 and len(configs.C5.mus()) == 256


def test_header_declares_exports_and_library_exports_them():
    hdr = open(os.path.join(os.path.dirname(__file__), "..", "include", "smpm_b200.h")).read()
    declared = set(re.findall(r"\b(smpm_[A-Za-z0-9_]+)\s*\(", hdr))
    assert declared == set(EXPORTS), declared ^ set(EXPORTS)
    lib = ctypes.CDLL(LIB_PATH)  # loads without a GPU; no compute calls here
    for name in EXPORTS:
        assert hasattr(lib, name), name


def test_oracle_golden_regression():
    g = np.load(os.path.join(GOLD, "c1_dbj.npz"))
    setup = O.build_poisson_setup(9, 4, 4, 1.0, 1.0, 2.0)
    f, _ = setup.prob.manufactured(4, False, 1234, 0)
    out = O.solve_poisson(setup, f, "dbj", 1e-10, 50, 50)
    assert out["res"].iterations == int(g["iterations"])
    assert np.linalg.norm(out["res"].x_S - g["x_S"]) <= 1e-12 * np.linalg.norm(g["x_S"])


def test_parity_pure_spectral_basis():
    """The z factor commutes with the reflection of the node index, and the
    product's spectral basis is built parity-pure from its even / odd blocks
    (fdm.StripFDM): every column of T (row of T^{-1}) is exactly even or odd,
    the modes are ordered pairs (even, odd) then reals (even, odd) — the
    structure the parity-split transform kernels detect (xformp.cuh) — and
    T diag T^{-1} still reproduces the operator."""
    from paper_1512_01756_b200.fdm import Geometry, StripFDM

    for n, m_z in ((6, 4), (9, 4), (11, 16)):
        geo = Geometry(n, 4, m_z, 4.0, 1.0)
        F = StripFDM(geo, device="cpu")
        w = geo.w
        J = np.eye(w)[::-1]
        assert np.abs(J @ F.Az @ J - F.Az).max() <= 1e-14 * np.abs(F.Az).max()
        npairs, T, Ti, rep = F.real_basis()
        assert np.abs(Ti @ T - np.eye(w)).max() < 1e-11
        par = []
        for m in range(w):
            even = np.array_equal(T[:, m], T[::-1, m]) and np.array_equal(Ti[m], Ti[m, ::-1])
            odd = np.array_equal(T[:, m], -T[::-1, m]) and np.array_equal(Ti[m], -Ti[m, ::-1])
            assert even != odd, m  # exactly one, bit for bit
            par.append(1 if even else -1)
        pp, pr = par[: 2 * npairs], par[2 * npairs:]
        assert pp == sorted(pp, reverse=True) and pr == sorted(pr, reverse=True)
        assert all(pp[2 * q] == pp[2 * q + 1] for q in range(npairs))
        assert par.count(1) == par.count(-1) == w // 2
        # the eigen-relation in the real basis: Az T = T B with B block diagonal (2x2 per pair)
        B = Ti @ F.Az @ T
        mask = np.zeros((w, w), dtype=bool)
        for q in range(npairs):
            mask[2 * q:2 * q + 2, 2 * q:2 * q + 2] = True
        for m in range(2 * npairs, w):
            mask[m, m] = True
        assert np.abs(B[~mask]).max() <= 1e-9 * np.abs(B).max()
