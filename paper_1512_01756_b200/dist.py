"""Mode sharding across ranks.

The Fourier modes are independent systems (proj/src/helmholtz.cpp:247-269),
so there is no collective inside a solve. Ranks own modes round-robin, which
spreads the slow low-wavenumber modes and puts the singular j = 0 system on
rank 0. After the solves, one all-gather over NVLink (NCCL; gloo on CPU in
the tests) collects per-mode results in mode order, and timings reduce by max.
"""
from __future__ import annotations


def shard_modes(nmodes: int, world: int, rank: int) -> list:
    """Modes owned by `rank`: m = rank, rank + world, ..."""
    return list(range(rank, nmodes, world))


def gather_modes(local, nmodes: int, world: int, group=None):
    """All-gather per-mode rows (local: tensor (n_local, ...) in this rank's
    mode order) into a (nmodes, ...) tensor in global mode order, on every rank."""
    import torch
    import torch.distributed as dist

    counts = [len(shard_modes(nmodes, world, r)) for r in range(world)]
    width = max(counts)
    pad = torch.zeros((width,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    out = torch.empty((nmodes,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    for r in range(world):
        out[r::world] = bufs[r][: counts[r]]
    return out


def max_over_ranks(values, device=None, group=None):
    """Element-wise max of a list of floats over ranks."""
    import torch
    import torch.distributed as dist

    t = torch.tensor(values, dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return t.tolist()
