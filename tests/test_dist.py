"""Multi-rank host logic with world_size 2 over gloo on CPU: mode sharding,
the all-gather of per-mode solutions into mode order, max-over-ranks
timing. Each rank solves its own modes with the CPU oracle standing in for
the device solve, and the gathered result must equal a single-process solve
of all modes."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1512_01756_b200.dist import gather_modes, max_over_ranks, mode_owners, shard_modes, stacked_norm


def test_shard_modes_partition():
    for nm in (1, 7, 128, 256):
        for ws in (1, 2, 4, 8):
            owned = sorted(m for r in range(ws) for m in shard_modes(nm, ws, r))
            assert owned == list(range(nm))
            assert 0 in shard_modes(nm, ws, 0)


def test_balanced_owners_partition_and_balance():
    """LPT on per-mode costs: a partition, mode 0 on rank 0, and the max per-rank
    load never above round-robin's on a C4-like skew (slow low modes)."""
    rng = np.random.default_rng(5)
    for nm in (5, 128, 256):
        costs = [40.0 / (1 + m) ** 0.5 + rng.uniform(0, 3) for m in range(nm)]
        for ws in (2, 4, 8):
            own = mode_owners(nm, ws, costs)
            assert sorted(m for o in own for m in o) == list(range(nm))
            assert 0 in own[0]
            lpt = max(sum(costs[m] for m in o) for o in own)
            rr = max(sum(costs[m] for m in o) for o in mode_owners(nm, ws))
            assert lpt <= rr + 1e-9
            assert own == mode_owners(nm, ws, list(costs))  # deterministic


def _solve_modes(modes):
    from oracle import oracle as O

    prob = O.Problem(6, 5, 3, 5.0, 1.0, 2.0)
    out = []
    for m in modes:
        mu = (2 * np.pi * m / 5.0) ** 2
        s = O.System(prob, mu, False)
        s.build_bj()
        f, _ = prob.manufactured(3, True, 1234, m, mu=mu)
        if mu == 0.0:
            u_S, u_L, _, _ = s.nullspace()
            s.build_coarse(u_S)
            b = O.project_out(s.schur_rhs(O.project_out(f, u_L)), u_S)
        else:
            s.build_coarse(None)
            b = prob.apply_B(prob.shifted_solve(mu, f))
        out.append(s.solve(b, "dbj", 1e-10, 100, 100).x_S)
    return np.array(out)


def _worker(rank, world, port, nmodes, result_path, costs=None):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = shard_modes(nmodes, world, rank, costs)
    x = torch.tensor(_solve_modes(mine))
    full = gather_modes(x, nmodes, world, costs=costs)
    tmax = max_over_ranks([float(rank + 1), float(10 - rank)])
    if rank == 0:
        np.save(result_path, full.numpy())
        np.save(result_path + ".t.npy", np.array(tmax))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_ranks(tmp_path):
    nmodes, world = 5, 2
    port = 29500 + (os.getpid() % 1000)
    path = str(tmp_path / "full.npy")
    mp.spawn(_worker, args=(world, port, nmodes, path), nprocs=world, join=True)
    full = np.load(path)
    ref = _solve_modes(list(range(nmodes)))
    assert full.shape == ref.shape
    assert np.array_equal(full, ref)  # identical CPU arithmetic per mode, gathered in mode order
    assert np.load(path + ".t.npy").tolist() == [2.0, 10.0]


def test_gloo_two_ranks_balanced(tmp_path):
    """The LPT assignment (skewed costs put modes 1 and 2 on different ranks out
    of round-robin order) gathers back into mode order as well."""
    nmodes, world = 5, 2
    costs = [5.0, 9.0, 8.0, 1.0, 1.0]
    assert mode_owners(nmodes, world, costs) != mode_owners(nmodes, world)
    port = 29700 + (os.getpid() % 1000)
    path = str(tmp_path / "full.npy")
    mp.spawn(_worker, args=(world, port, nmodes, path, costs), nprocs=world, join=True)
    full = np.load(path)
    ref = _solve_modes(list(range(nmodes)))
    assert np.array_equal(full, ref)


def _norm_worker(rank, world, port, path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(11)
    v = rng.standard_normal((5, 40))
    mine = shard_modes(5, world, rank)
    n = stacked_norm([float(v[m] @ v[m]) for m in mine])
    np.save(f"{path}.{rank}.npy", np.array([n, float(np.sqrt((v * v).sum()))]))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_stacked_norm(tmp_path):
    """The stacked right-hand-side norm over mode-sharded ranks (the reduction the
    stacked solve's all-reduce hook performs per inner product): identical on
    both ranks and equal to the single-process norm."""
    port = 29900 + (os.getpid() % 1000)
    path = str(tmp_path / "n")
    mp.spawn(_norm_worker, args=(2, port, path), nprocs=2, join=True)
    a, b = np.load(path + ".0.npy"), np.load(path + ".1.npy")
    assert a[0] == b[0]
    assert abs(a[0] - a[1]) <= 1e-14 * a[1]
