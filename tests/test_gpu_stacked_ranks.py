"""Stacked 3D solve across ranks (smpm_batch_set_allreduce): the stack's modes are
split over two batches ("ranks") that iterate together, every inner product
summed over both through the all-reduce hook.  One GPU stands in for two: each
rank is a host thread with its own context and stream, and the hook is a HOST
rendezvous (stream sync, sum in rank order, write back) — no kernel waits on
another.  The split solve must reproduce the single-batch stacked solve:
identical iteration counts, solutions to rounding."""
import threading

import numpy as np
import pytest

from tests._cases import build_case, gpu_batch

pytestmark = pytest.mark.gpu


class HostRendezvous:
    """In-process sum all-reduce between `world` threads (deterministic rank order)."""

    def __init__(self, world):
        self.world = world
        self.bar = threading.Barrier(world)
        self.parts = [None] * world
        self.calls = 0

    def hook(self, rank):
        import torch

        def fn(ptr, count, stream):
            from paper_1512_01756_b200.dist import _DevPtr

            buf = torch.as_tensor(_DevPtr(ptr, count), device="cuda")
            s = torch.cuda.ExternalStream(stream) if stream else torch.cuda.current_stream()
            s.synchronize()
            self.parts[rank] = buf.cpu().numpy().copy()
            self.bar.wait()
            tot = self.parts[0].copy()
            for r in range(1, self.world):
                tot = tot + self.parts[r]
            self.bar.wait()
            with torch.cuda.stream(s):
                buf.copy_(torch.tensor(tot, device="cuda"))
            s.synchronize()
            if rank == 0:
                self.calls += 1

        return fn


@pytest.mark.parametrize("method,restart", [("dbj", 0), ("dbj", 4), ("2las", 0)])
def test_stacked_two_ranks_match_single(method, restart):
    import torch

    from paper_1512_01756_b200 import Context

    mus = [(2 * np.pi * j / 6.0) ** 2 for j in range(6)]
    case = build_case(7, 6, 4, 6.0, 1.0, mus, kmax=4, decay=True)
    ctx = Context(0)
    full = gpu_batch(ctx, case, spectral=True)
    bS = torch.tensor(case.b_S, device="cuda")
    ref = full.solve_stacked(bS, method, 1e-10, 60, restart)
    torch.cuda.synchronize()

    owners = [[0, 2, 4], [1, 3, 5]]
    rv = HostRendezvous(2)
    out = [None, None]
    err = [None, None]

    def run(rank):
        try:
            from tests._cases import Case

            sub = Case(case.prob, [case.systems[i] for i in owners[rank]], [mus[i] for i in owners[rank]],
                       case.b_S[owners[rank]], case.u_S, case.u_L, [case.kinds[i] for i in owners[rank]])
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                b = gpu_batch(Context(0), sub, spectral=True)
                b.set_allreduce(rv.hook(rank))
                res = b.solve_stacked(torch.tensor(sub.b_S, device="cuda"), method, 1e-10, 60, restart)
                st.synchronize()
            out[rank] = res
        except Exception as e:  # a failing rank must not leave the other at the barrier
            err[rank] = e
            rv.bar.abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert err == [None, None], err
    assert rv.calls > 3 * ref.iterations[0]  # norms + three reductions per Arnoldi step
    for rank in range(2):
        res = out[rank]
        assert res.iterations[0] == ref.iterations[0], (res.iterations, ref.iterations)
        assert res.converged[0] == ref.converged[0]
        assert abs(res.final_rel_residual[0] - ref.final_rel_residual[0]) <= 1e-6 * max(ref.final_rel_residual[0], 1e-12) + 1e-14
        x = res.x_S.cpu().numpy()
        xr = ref.x_S.cpu().numpy()[owners[rank]]
        for i, m in enumerate(owners[rank]):
            a, c = x[i], xr[i]
            if mus[m] == 0.0:
                a, c = a - a.mean(), c - c.mean()
            assert np.linalg.norm(a - c) <= 1e-9 * np.linalg.norm(c), (rank, i)
