"""Device-side per-mode setup (smpm_batch_set_fdm): the library
builds every system's spectral diagonals, dense couplings, block-Jacobi inverses,
strip row sums and coarse matrix with its own kernels from the geometry-level
fast-diagonalisation factors.  Held against the host setup of the same problem
(dense couplings from fdm.py, LU block inverses through cuSOLVER), which the
parity tests hold to the oracle: operators to 1e-11, coarse matrices to 1e-12,
identical iteration counts, solutions to the conditioning-limited level."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,m_x,m_z", [(8, 5, 2), (8, 4, 6), (11, 6, 16), (17, 5, 16)])
def test_device_setup_matches_host_setup(ctx, n, m_x, m_z):
    import torch

    from paper_1512_01756_b200.configs import Config
    from paper_1512_01756_b200.problems import build_problem, load_batch

    cfg = Config(f"w{n * m_z}", n, m_x, m_z, float(m_x), 1.0, 4, True, 100, modes=6, l_y=float(m_x))
    host = build_problem(cfg, device="cuda")
    dev = build_problem(cfg, device="cuda", device_setup=True)
    assert dev.GW is None
    dev.b_S = host.b_S
    bh = load_batch(ctx, host)
    bd = load_batch(ctx, dev)
    assert bd.query("spectral") == 1
    gen = torch.Generator(device="cuda").manual_seed(7)
    v = torch.randn((len(host.mus), bh.k), device="cuda", dtype=torch.float64, generator=gen)

    def close(a, b, tol):
        num = torch.linalg.norm(a - b, dim=1)
        den = torch.linalg.norm(b, dim=1)
        assert float((num / den).max()) <= tol, float((num / den).max())

    close(bd.apply_S(v), bh.apply_S(v), 1e-11)
    close(bd.apply_St(v), bh.apply_St(v), 1e-11)
    close(bd.apply_block_jacobi_inv(v), bh.apply_block_jacobi_inv(v), 1e-9)
    close(bd.apply_P(v, fused=True), bh.apply_P(v, fused=True), 1e-10)
    close(bd.apply_P(v, fused=False), bh.apply_P(v, fused=False), 1e-10)
    Ch, th, sh = bh.coarse_info()
    Cd, td, sd = bd.coarse_info()
    assert list(th) == list(td) and list(sh) == list(sd)
    assert np.abs(Cd - Ch).max() <= 1e-11 * np.abs(Ch).max()
    bS = torch.tensor(host.b_S, device="cuda")
    for method in ("dbj", "2las"):
        rh = bh.solve(bS, method, 1e-10, 100, 0)
        rd = bd.solve(bS, method, 1e-10, 100, 0)
        assert all(rd.converged)
        assert max(abs(a - c) for a, c in zip(rh.iterations, rd.iterations)) <= 1
        th_ = bh.solve(bS, method, 1e-14, 100, 0).x_S.cpu().numpy()
        td_ = bd.solve(bS, method, 1e-14, 100, 0).x_S.cpu().numpy()
        for i, mu in enumerate(host.mus):
            a, c = th_[i], td_[i]
            if mu == 0.0:
                a, c = a - a.mean(), c - c.mean()
            assert np.linalg.norm(a - c) <= 2e-8 * np.linalg.norm(a), (method, i)
    # the device right-hand sides go through the stored strip factors as well
    dev2 = build_problem(cfg, device="cuda", device_setup=True, device_rhs=True)
    load_batch(ctx, dev2)
    for i in range(len(host.mus)):
        assert np.linalg.norm(dev2.b_S[i] - host.b_S[i]) <= 1e-9 * np.linalg.norm(host.b_S[i]), i


def test_device_setup_rejects_unaligned_width(ctx):
    from paper_1512_01756_b200 import SchurBatch
    from paper_1512_01756_b200._lib import SmpmError
    from paper_1512_01756_b200.fdm import Geometry, StripFDM

    geo = Geometry(5, 4, 3, 4.0, 1.0)  # w = 15
    F = StripFDM(geo, device="cpu")
    npairs, T, Ti, _ = F.real_basis()
    b = SchurBatch(ctx, 5, 4, 3, 1)
    with pytest.raises(SmpmError):
        b.set_fdm(npairs, T, Ti, F.strip_factors([1.0]))


@pytest.mark.slow
def test_device_setup_at_c5_scale(ctx):
    """The bench's own setup path at C5 size (w = 544, k = 277,440; modes 0, 3, 8,
    255): operators of the device-built batch against the host-built one (which
    test_gpu_parity / test_gpu_configs hold to the oracle), the singular mode's
    compatibility, and solves whose true residual is at the tolerance."""
    import torch

    from paper_1512_01756_b200 import configs
    from paper_1512_01756_b200.problems import build_problem, load_batch

    cfg = configs.C5
    modes = [0, 3, 8, 255]
    host = build_problem(cfg, modes, device="cuda", device_rhs=True)
    dev = build_problem(cfg, modes, device="cuda", device_rhs=True, device_setup=True)
    bh = load_batch(ctx, host)
    bd = load_batch(ctx, dev)
    gen = torch.Generator(device="cuda").manual_seed(3)
    v = torch.randn((len(modes), bh.k), device="cuda", dtype=torch.float64, generator=gen)

    def close(a, b, tol):
        r = torch.linalg.norm(a - b, dim=1) / torch.linalg.norm(b, dim=1)
        assert float(r.max()) <= tol, float(r.max())

    close(bd.apply_S(v), bh.apply_S(v), 1e-10)
    close(bd.apply_block_jacobi_inv(v), bh.apply_block_jacobi_inv(v), 1e-8)
    close(bd.apply_P(v, fused=True), bh.apply_P(v, fused=True), 1e-9)
    for i in range(len(modes)):
        assert np.linalg.norm(dev.b_S[i] - host.b_S[i]) <= 1e-10 * np.linalg.norm(host.b_S[i]), i
    bS = torch.tensor(dev.b_S, device="cuda")
    res = bd.solve(bS, "dbj", 1e-10, 400, 0, history=False)
    assert all(res.converged)
    r = bd.apply_S(res.x_S) - bS
    assert float((torch.linalg.norm(r, dim=1) / torch.linalg.norm(bS, dim=1)).max()) < 1e-9


@pytest.mark.parametrize("m_x", [2, 3, 4])
def test_device_setup_block_edges(ctx, m_x):
    """d = 1 (a single one-interface block, no strip solver), d = 2 (first == last
    block) and d = 3 (a full block plus the trailing single one): the device-built
    pool against the host-built one."""
    import torch

    from paper_1512_01756_b200.configs import Config
    from paper_1512_01756_b200.problems import build_problem, load_batch

    cfg = Config(f"edge{m_x}", 8, m_x, 4, 1.5 * m_x, 1.0, 3, True, 100, modes=3, l_y=3.0)
    host = build_problem(cfg, [1, 2], device="cuda")
    dev = build_problem(cfg, [1, 2], device="cuda", device_setup=True)
    dev.b_S = host.b_S
    bh, bd = load_batch(ctx, host), load_batch(ctx, dev)
    gen = torch.Generator(device="cuda").manual_seed(11)
    v = torch.randn((2, bh.k), device="cuda", dtype=torch.float64, generator=gen)
    for op in ("apply_S", "apply_block_jacobi_inv"):
        a, c = getattr(bd, op)(v), getattr(bh, op)(v)
        rel = float((torch.linalg.norm(a - c, dim=1) / torch.linalg.norm(c, dim=1)).max())
        assert rel <= 1e-10, (op, rel)
    bS = torch.tensor(host.b_S, device="cuda")
    rh, rd = bh.solve(bS, "dbj", 1e-10, 100, 0), bd.solve(bS, "dbj", 1e-10, 100, 0)
    assert all(rd.converged) and max(abs(a - c) for a, c in zip(rh.iterations, rd.iterations)) <= 1
