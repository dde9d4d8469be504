"""The end-to-end entry point (smpm_solve_host: host b_S in, host x_S out, the
copies inside the call) against the device-pointer solve of the same batch:
identical reports and bitwise-identical x_S, whichever way the epilogue is split
(early epilogue of the stopped systems with their rows copied out while the rest
iterate — before the grid tail, or, without a tail, once an eighth of the systems
is left — or one epilogue at the end)."""
import numpy as np
import pytest

from tests._cases import build_case, gpu_batch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("grid,early", [(1, 1), (0, 1), (0, 0), (1, 0)])
def test_solve_host_matches_device_solve(ctx, grid, early):
    import torch

    # 24 Helmholtz modes: the low ones need 3-4x the iterations of the rest, so the
    # early epilogue triggers in both paths
    mus = [(2 * np.pi * j / 8.0) ** 2 for j in range(24)]
    case = build_case(7, 8, 4, 8.0, 1.0, mus, kmax=4, decay=True)
    b = gpu_batch(ctx, case, spectral=True)
    b.tune(grid=grid, early=early)
    ref = b.solve(torch.tensor(case.b_S, device="cuda"), "dbj", 1e-10, 100, 0)
    its = list(ref.iterations)
    assert max(its) >= 2 * sorted(its)[len(its) // 2]  # a real spread of stopping times
    hb = torch.tensor(case.b_S).pin_memory()
    hx = torch.empty_like(hb).pin_memory()
    res = b.solve_host(hb.numpy(), "dbj", 1e-10, 100, 0, "cgs2", True, out=hx.numpy())
    torch.cuda.synchronize()
    assert list(res.iterations) == its
    assert list(res.converged) == list(ref.converged)
    assert np.array_equal(hx.numpy(), ref.x_S.cpu().numpy())
    # pageable host memory works as well
    out2 = np.empty_like(case.b_S)
    b.solve_host(np.ascontiguousarray(case.b_S), "dbj", 1e-10, 100, 0, "cgs2", True, out=out2)
    assert np.array_equal(out2, ref.x_S.cpu().numpy())


def test_prefetched_rhs_matches_plain_solve_host(ctx):
    """smpm_prefetch_rhs: uploads started ahead of their solve_host (two outstanding,
    the same pinned buffer reused as in bench.py, and two different buffers) give the
    same x_S bit for bit as solve_host copying by itself."""
    import torch

    mus = [(2 * np.pi * j / 8.0) ** 2 for j in range(10)]
    case = build_case(7, 8, 4, 8.0, 1.0, mus, kmax=4, decay=True)
    b = gpu_batch(ctx, case, spectral=True)
    h1 = torch.tensor(case.b_S).pin_memory()
    h2 = (2.0 * torch.tensor(case.b_S)).pin_memory()
    out = torch.empty_like(h1).pin_memory()
    ref1 = b.solve_host(h1.numpy(), "dbj", 1e-10, 100, 0, "cgs2", True).x_S.copy()
    ref2 = b.solve_host(h2.numpy(), "dbj", 1e-10, 100, 0, "cgs2", True).x_S.copy()
    a1, a2 = h1.numpy(), h2.numpy()
    b.prefetch_rhs(a1)
    for _ in range(3):  # steady state: next upload first, then the solve of the older one
        b.prefetch_rhs(a1)
        b.solve_host(a1, "dbj", 1e-10, 100, 0, "cgs2", True, out=out.numpy())
        assert np.array_equal(out.numpy(), ref1)
    b.solve_host(a1, "dbj", 1e-10, 100, 0, "cgs2", True, out=out.numpy())  # consumes the last upload
    assert np.array_equal(out.numpy(), ref1)
    b.prefetch_rhs(a1)
    b.prefetch_rhs(a2)
    b.solve_host(a2, "dbj", 1e-10, 100, 0, "cgs2", True, out=out.numpy())
    assert np.array_equal(out.numpy(), ref2)
    b.solve_host(a1, "dbj", 1e-10, 100, 0, "cgs2", True, out=out.numpy())
    assert np.array_equal(out.numpy(), ref1)
