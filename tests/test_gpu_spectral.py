"""Spectral operator path (spectral.cuh) vs the oracle: the same parity bar as
the dense path (solution 1e-10 or conditioning-aware, iterations +-1,
histories), on geometries whose z eigenbasis has complex-conjugate pairs, in
batches small enough for the grid-persistent tail and large enough for the
per-stage kernels."""
import numpy as np
import pytest

from tests._cases import build_case, gpu_batch
from tests.test_gpu_solve import check_solve

pytestmark = pytest.mark.gpu


def _pairs(case):
    from tests._cases import spectral_factors

    return spectral_factors(case)[0]


@pytest.mark.parametrize("method", ["dbj", "bj", "schur", "2las"])
def test_spectral_small(ctx, method):
    case = build_case(6, 6, 4, 24.0, 4.0, (0.0,))
    b = gpu_batch(ctx, case, spectral=True)
    check_solve(case, b, method, max_iter=200)


def test_spectral_c1(ctx):
    case = build_case(9, 4, 4, 1.0, 1.0, (0.0,), kmax=4, decay=False)
    assert _pairs(case) > 0  # the complex-pair branch is exercised
    b = gpu_batch(ctx, case, spectral=True)
    check_solve(case, b, "dbj", max_iter=50)
    check_solve(case, b, "dbj", max_iter=50, fused=False)


@pytest.mark.parametrize("m_x", [2, 3, 4, 5])
def test_spectral_block_edges(ctx, m_x):
    # d = 1 (single block only), d = 2 (first == last block), odd / even d
    mus = [0.0, (2 * np.pi / 3.0) ** 2]
    case = build_case(6, m_x, 4, 1.5 * m_x, 1.0, mus, kmax=3, decay=True)
    b = gpu_batch(ctx, case, spectral=True)
    check_solve(case, b, "dbj", max_iter=120)
    if m_x > 3:  # for d <= 2 one block is all of the singular S: plain BJ is ill-posed
        check_solve(case, b, "bj", max_iter=120)


def test_spectral_helmholtz_batch(ctx):
    # 40 modes: per-stage kernels for the wide phase, grid tail for the rest
    mus = [(2 * np.pi * j / 6.0) ** 2 for j in range(40)]
    case = build_case(7, 6, 4, 6.0, 1.0, mus, kmax=4, decay=True)
    b = gpu_batch(ctx, case, spectral=True)
    check_solve(case, b, "dbj", max_iter=100)


def test_spectral_matches_dense(ctx):
    # the two operator forms of the same batch agree to rounding
    import torch

    mus = [(2 * np.pi * j / 6.0) ** 2 for j in range(12)]
    case = build_case(7, 9, 4, 9.0, 1.0, mus, kmax=4, decay=True)
    bd = gpu_batch(ctx, case)
    bs = gpu_batch(ctx, case, spectral=True)
    rhs = torch.tensor(case.b_S, device="cuda")
    rd = bd.solve(rhs, "dbj", 1e-10, 100, 0, "cgs2", True)
    rs = bs.solve(rhs, "dbj", 1e-10, 100, 0, "cgs2", True)
    assert max(abs(a - c) for a, c in zip(rd.iterations, rs.iterations)) <= 1
    xd, xs = rd.x_S.cpu().numpy(), rs.x_S.cpu().numpy()
    for i in range(len(mus)):
        a, c = xd[i], xs[i]
        if mus[i] == 0.0:
            a, c = a - a.mean(), c - c.mean()
        assert np.linalg.norm(a - c) <= 1e-8 * np.linalg.norm(a), i


def test_spectral_odd_w_falls_back(ctx):
    # odd w has no 16-byte aligned transform plan: the dense path runs
    case = build_case(5, 4, 3, 4.0, 1.0, (0.0,))
    b = gpu_batch(ctx, case, spectral=True)
    check_solve(case, b, "dbj", max_iter=100)
