"""Batch sharding across ranks: independent simulations are split over the
ranks of a torch.distributed group; nothing is exchanged per time step.  The only collectives are one
all-gather of per-sim results at the end of a run and the max-over-ranks of the measured device time.

Host-side logic only (no kernels); covered by a world_size-2 gloo test on CPU.
"""
from __future__ import annotations


def shard_range(n_sims: int, world: int, rank: int):
    """Contiguous block [lo, hi) of the sims owned by `rank` (sizes differ by at most one)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(n_sims, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def shared_youngs_ref(youngs_all) -> float:
    """Young's modulus of the one factorised A for a batched run: the max over the
    WHOLE batch, computed before sharding, so iterates do not depend on the GPU count."""
    return float(max(youngs_all))


def gather_rows(local, world: int, group=None):
    """All-gather per-sim result rows (a [n_local, ...] tensor) into the full [n_sims, ...] tensor in rank
    order.  Ranks may own different counts; rows are padded to the largest shard for the collective."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return local
    n = torch.tensor([local.shape[0]], dtype=torch.int64, device=local.device)
    counts = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(counts, n, group=group)
    counts = [int(c.item()) for c in counts]
    m = max(counts)
    pad = torch.zeros((m,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    bufs = [torch.zeros_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    return torch.cat([b[:c] for b, c in zip(bufs, counts)], 0)


def max_over_ranks(value: float, world: int, device=None) -> float:
    """Max of a per-rank scalar (the timed region's device milliseconds)."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
