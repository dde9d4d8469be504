"""Mode sharding across ranks.

The Fourier modes are independent systems (proj/src/helmholtz.cpp:247-269),
so there is no collective inside a solve. Ranks own modes round-robin by
default, which spreads the slow low-wavenumber modes and puts the singular
j = 0 system on rank 0; with per-mode cost estimates (e.g. the iteration
counts of an earlier solve of the same batch) the modes are instead assigned
longest-first to the least-loaded rank (LPT), which evens out the per-rank
time when a few slow modes dominate. After the solves, one all-gather over
NVLink (NCCL; gloo on CPU in the tests) collects per-mode results in mode
order, and timings reduce by max.
"""
from __future__ import annotations


def mode_owners(nmodes: int, world: int, costs=None) -> list:
    """Mode lists of every rank: round-robin without costs, else LPT on `costs`
    (ties broken by mode index, then rank index: deterministic on every rank).
    Each list is ascending; mode 0 always lives on rank 0."""
    if costs is None:
        return [list(range(r, nmodes, world)) for r in range(world)]
    if len(costs) != nmodes:
        raise ValueError("one cost per mode")
    load = [0.0] * world
    owners = [[] for _ in range(world)]
    owners[0].append(0)
    load[0] += float(costs[0])
    for m in sorted(range(1, nmodes), key=lambda q: (-float(costs[q]), q)):
        r = min(range(world), key=lambda q: (load[q], q))
        owners[r].append(m)
        load[r] += float(costs[m])
    return [sorted(o) for o in owners]


def shard_modes(nmodes: int, world: int, rank: int, costs=None) -> list:
    """Modes owned by `rank` (mode_owners)."""
    return mode_owners(nmodes, world, costs)[rank]


def gather_modes(local, nmodes: int, world: int, group=None, costs=None):
    """All-gather per-mode rows (local: tensor (n_local, ...) in this rank's
    mode order) into a (nmodes, ...) tensor in global mode order, on every rank.
    `costs` must be the same as the sharding's."""
    import torch
    import torch.distributed as dist

    owners = mode_owners(nmodes, world, costs)
    width = max(len(o) for o in owners)
    pad = torch.zeros((width,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    out = torch.empty((nmodes,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    for r in range(world):
        if owners[r]:
            out[torch.tensor(owners[r], device=local.device)] = bufs[r][: len(owners[r])]
    return out


def max_over_ranks(values, device=None, group=None):
    """Element-wise max of a list of floats over ranks."""
    import torch
    import torch.distributed as dist

    t = torch.tensor(values, dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return t.tolist()


class _DevPtr:
    """A device buffer of `count` doubles as a zero-copy torch view (__cuda_array_interface__)."""

    def __init__(self, ptr: int, count: int):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": "<f8", "data": (ptr, False), "version": 3,
                                         "strides": None}


def allreduce_hook(group=None):
    """All-reduce hook for SchurBatch.set_allreduce: the stacked solve's inner
    products summed over the ranks of `group` (NCCL over NVLink on GPUs), one
    all-reduce per inner product (proj/src/helmholtz.cpp:187-246 across GPUs).

    The library passes its own device buffer and the stream its kernels run on;
    torch's NCCL all_reduce orders itself after the current stream's work and
    makes the current stream wait for the result, so the hook runs it under
    that stream.  NCCL leaves bitwise-identical sums on every rank, which the
    stacked solve relies on (all ranks take the same stopping decisions)."""
    import torch
    import torch.distributed as dist

    def hook(ptr: int, count: int, stream: int):
        buf = torch.as_tensor(_DevPtr(ptr, count), device="cuda")
        ext = torch.cuda.ExternalStream(stream) if stream else torch.cuda.current_stream()
        with torch.cuda.stream(ext):
            dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)

    return hook


def stacked_norm(local_sq, group=None):
    """sqrt of the sum over ranks of a rank's partial squared norms (host helper
    for callers assembling the stacked right-hand-side norm themselves)."""
    import torch
    import torch.distributed as dist

    t = torch.as_tensor(local_sq, dtype=torch.float64).sum().reshape(1).clone()
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return float(t.sqrt())
