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


@pytest.mark.parametrize("n,m_z", [(17, 16), (13, 32), (17, 32)])
def test_spectral_large_w(ctx, n, m_z):
    """w = 272 / 416 / 544 (the C3 / C2 / C5 interface widths): the transforms run
    on the K-streamed kernel (xformk.cuh) in the per-stage path (12 live systems)
    and in the strip solves.  The spectral solves hold the oracle's bars on the
    same couplings (tests/test_gpu_parity.py envelope), and the device b_S
    (schur_rhs through the streamed transform) matches the host FDM."""
    import torch

    from paper_1512_01756_b200.configs import Config
    from paper_1512_01756_b200.problems import build_problem, load_batch
    from tests.test_gpu_parity import compare_modes, oracle_systems, perturbed, run_jobs

    cfg = Config(f"w{n * m_z}", n, 4, m_z, 4.0, 1.0, 4, True, 100, modes=12, l_y=4.0)
    ps = build_problem(cfg, device="cuda")
    bs = load_batch(ctx, ps)
    rhs = torch.tensor(ps.b_S, device="cuda")
    rs = bs.solve(rhs, "dbj", 1e-10, 100, 0)
    _, systems = oracle_systems(ps)
    ns = len(systems)
    rr = [ps.b_S, perturbed(ps.b_S, 1), perturbed(ps.b_S, 2)]
    out = run_jobs([(systems[i], r[i], "dbj", 1e-10, 100) for r in rr for i in range(ns)])
    rows, fails = compare_modes(rs, ps, out[:ns], [[out[ns + i], out[2 * ns + i]] for i in range(ns)],
                                systems=systems)
    assert not fails, fails
    assert all(rs.converged)
    dev = build_problem(cfg, device="cuda", device_rhs=True)
    load_batch(ctx, dev)
    for i in range(len(ps.mus)):
        assert np.linalg.norm(dev.b_S[i] - ps.b_S[i]) <= 1e-9 * np.linalg.norm(ps.b_S[i]), i


@pytest.mark.parametrize("n,m_z", [(8, 2), (8, 6), (11, 16), (17, 16), (13, 32), (17, 32)])
def test_parity_split_transforms(ctx, n, m_z):
    """The parity-split transform kernels (xformp.cuh: two h x h contractions with
    the fold / unfold inside the kernel) against the full w x w transform kernels
    on the same batch, w = 16 ... 544 (every template instance): the strip solves
    (schur_rhs = T^{-1}, per-mode, T on all strip rows) agree to rounding, and so do
    the solves (same iteration counts +-1 at rtol 1e-10; x_S of the iterates driven
    to the rounding floor to 2e-8 of the solution scale)."""
    import torch

    from paper_1512_01756_b200.configs import Config
    from paper_1512_01756_b200.problems import build_problem, load_batch

    cfg = Config(f"w{n * m_z}", n, 5, m_z, 5.0, 1.0, 4, True, 100, modes=12, l_y=5.0)
    ps = build_problem(cfg, device="cuda", device_rhs=True)
    f = ps.f.clone()
    out = {}
    for mode in (0, 2):
        ps.b_S, ps.f = None, f.clone()
        b = load_batch(ctx, ps)
        b.tune(xform_parity=mode)
        bS = b.schur_rhs(ps.f)
        res = b.solve(bS, "dbj", 1e-10, 100, 0, history=False)
        # the solutions are compared on iterates driven to the rounding floor: two
        # rtol-1e-10 iterates differ by 1e-8 of the solution scale at these condition numbers
        tight = b.solve(bS, "dbj", 1e-14, 100, 0, history=False)
        torch.cuda.synchronize()
        out[mode] = (bS.cpu().numpy(), tight.x_S.cpu().numpy(), list(res.iterations), list(res.converged))
    b0, x0, it0, cv0 = out[0]
    b2, x2, it2, cv2 = out[2]
    assert all(cv0) and all(cv2)
    for i in range(len(ps.mus)):
        assert np.linalg.norm(b2[i] - b0[i]) <= 1e-12 * np.linalg.norm(b0[i]), i
        a, c = x0[i], x2[i]
        if ps.mus[i] == 0.0:
            a, c = a - a.mean(), c - c.mean()
        assert np.linalg.norm(a - c) <= 2e-8 * np.linalg.norm(a), i
    assert max(abs(a - c) for a, c in zip(it0, it2)) <= 1


@pytest.mark.parametrize("method", ["dbj", "2las", "bj"])
def test_per_mode_pass_variants_agree(ctx, method):
    """The three per-mode pass kernels — spec_op3 (16 bytes per lane: a pair or two
    real modes, default), spec_op2 (one mode per lane), spec_op (staged) — run the
    same per-mode arithmetic: same iteration counts, solutions to rounding; each
    also holds the oracle's bars (check_solve on the default)."""
    import torch

    mus = [(2 * np.pi * j / 6.0) ** 2 for j in range(20)]
    case = build_case(9, 7, 4, 7.0, 1.0, mus, kmax=4, decay=True)
    assert _pairs(case) > 0
    b = gpu_batch(ctx, case, spectral=True)
    b.tune(grid=0)
    check_solve(case, b, method, max_iter=100)
    rhs = torch.tensor(case.b_S, device="cuda")
    out = {}
    for v in (2, 1, 0):
        b.tune(spec_v2=v)
        r = b.solve(rhs, method, 1e-10, 100, 0)
        out[v] = (list(r.iterations), r.x_S.cpu().numpy())
    for v in (1, 0):
        assert max(abs(a - c) for a, c in zip(out[2][0], out[v][0])) <= 1, v
        for i in range(len(mus)):
            a, c = out[2][1][i], out[v][1][i]
            if mus[i] == 0.0:
                a, c = a - a.mean(), c - c.mean()
            assert np.linalg.norm(a - c) <= 1e-8 * np.linalg.norm(a), (v, i)
