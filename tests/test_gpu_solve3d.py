"""The 3D Fourier-extended solve (solve_3d, /root/reference/proj/src/helmholtz.cpp:150-297)
on the device against a restatement built from the oracle's pieces: the transverse
transforms against proj/src/fourier.cpp:47-86 (restated with numpy), the per-mode right-hand
sides, solves and recoveries against the oracle's LU / real-Schur strip solves and
deflated GMRES."""
import math

import numpy as np
import pytest

from oracle import oracle as O
from paper_1512_01756_b200 import Context  # noqa: F401
from paper_1512_01756_b200.solve3d import Fourier3D, fourier_y, inverse_fourier_y

pytestmark = pytest.mark.gpu


def np_fourier_y(field):
    """proj/src/fourier.cpp:47-62: first m_y/2 forward DFT coefficients / m_y, per row."""
    m = field.shape[0]
    return np.fft.fft(field, axis=0)[: m // 2] / m


def np_inverse_fourier_y(coeff, m):
    """proj/src/fourier.cpp:64-86: Hermitian extension (Nyquist zero), +1 transform, real part."""
    half = m // 2
    row = np.zeros((m, coeff.shape[1]), dtype=complex)
    row[0] = coeff[0]
    for j in range(1, half):
        row[j] = coeff[j]
        row[m - j] = np.conj(coeff[j])
    return (np.fft.ifft(row, axis=0) * m).real


@pytest.mark.parametrize("m_y", [2, 8, 32, 64, 128, 256, 512, 1024])
def test_fourier_transforms(ctx, m_y):
    import torch

    r = 1000
    f = np.random.default_rng(3).standard_normal((m_y, r))
    c = fourier_y(torch.tensor(f, device="cuda"), m_y).cpu().numpy()
    ref = np_fourier_y(f)
    assert np.abs(c[0::2] - ref.real).max() < 1e-14 * np.abs(f).max() * 4
    assert np.abs(c[1::2] - ref.imag).max() < 1e-14 * np.abs(f).max() * 4
    u = inverse_fourier_y(torch.tensor(c, device="cuda"), m_y).cpu().numpy()
    uref = np_inverse_fourier_y(ref, m_y)
    assert np.abs(u - uref).max() < 1e-13 * max(1.0, np.abs(uref).max())


def oracle_solve_3d(prob, f, m_y, l_y, tol=1e-10, max_iter=100):
    """solve_3d's independent branch (proj/src/helmholtz.cpp:150-297) from oracle pieces."""
    half = m_y // 2
    fh = np_fourier_y(f)  # (half, r) complex
    s0 = O.System(prob, 0.0, False)
    s0.build_bj()
    u_S, u_L, _, _ = s0.nullspace()
    s0.build_coarse(u_S)
    uh = np.zeros_like(fh)
    for j in range(half):
        mu = (2 * math.pi * j / l_y) ** 2
        parts = []
        for p in range(2):
            fj = fh[j].real.copy() if p == 0 else fh[j].imag.copy()
            if j == 0:
                fj = O.project_out(fj, u_L)
                b = O.project_out(s0.schur_rhs(fj), u_S)
                x = s0.solve(b, "dbj", tol, max_iter, 0).x_S
                parts.append(prob.solve_A(fj - prob.apply_E(x)))
            else:
                s = O.System(prob, mu, False)
                s.build_bj()
                s.build_coarse(None)
                b = prob.apply_B(prob.shifted_solve(mu, fj))
                x = s.solve(b, "dbj", tol, max_iter, 0).x_S
                parts.append(prob.shifted_solve(mu, fj - prob.apply_E(x)))
        uh[j] = parts[0] + 1j * parts[1]
    return np_inverse_fourier_y(uh, m_y)


@pytest.mark.parametrize("stacked", [False, True])
def test_solve_3d_small(ctx, stacked):
    import torch

    n, m_x, m_z, l_x, l_z, m_y, l_y = 7, 5, 4, 5.0, 1.0, 8, 2.0
    prob = O.Problem(n, m_x, m_z, l_x, l_z, 2.0)
    r = prob.r
    # seeded smooth 3D forcing: cosine modes in x, z times a few transverse harmonics
    x, z = prob.coords()
    rng = np.random.default_rng(1234)
    y = np.arange(m_y) * l_y / m_y
    f = np.zeros((m_y, r))
    for _ in range(6):
        kx, kz, ky = rng.integers(0, 4), rng.integers(0, 3), rng.integers(0, m_y // 2)
        a, ph = rng.standard_normal(), rng.uniform(0, 2 * math.pi)
        f += a * np.cos(kx * math.pi * (x + l_x / 2) / l_x)[None, :] * np.cos(kz * math.pi * (z + l_z / 2) / l_z)[None, :] \
            * np.cos(2 * math.pi * ky * y / l_y + ph)[:, None]
    solver = Fourier3D(ctx, n, m_x, m_z, l_x, l_z, m_y, l_y)
    res = solver.solve(torch.tensor(f, device="cuda"), "dbj", 1e-10, 100, stacked=stacked)
    assert all(res.converged) and res.rel_residual < 1e-9
    u = res.u.cpu().numpy()
    uref = oracle_solve_3d(prob, f, m_y, l_y)
    # the Neumann j = 0 mode fixes u up to a constant (proj/src/bench.cpp:358-360): mean-removed
    d = (u - u.mean()) - (uref - uref.mean())
    assert np.linalg.norm(d) < 1e-8 * np.linalg.norm(uref - uref.mean())
