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


def shared_youngs_ref(youngs_all, accel: bool = False) -> float:
    """Young's modulus of the one factorised A for a batched run, computed over the WHOLE
    batch before sharding, so iterates do not depend on the GPU count: the batch max (the majorising A_ref of
    plain PD) or, with the quasi-Newton forward/adjoint (A_ref^{-1} only preconditions), the geometric mean of
    the batch extremes."""
    import math
    E = [float(e) for e in youngs_all]
    return math.sqrt(min(E) * max(E)) if accel else max(E)


PER_SIM_KEYS = ("q0", "v0", "f_ext", "youngs", "act", "c_q", "c_v", "tip_target")


def shard_inputs(inp, world: int, rank: int, accel: bool = True):
    """The slice [lo, hi) of a pd_inputs workload owned by `rank`: per-sim arrays cut along the batch, the
    mesh and lists shared, and `youngs_ref` fixed from the whole batch (so a sim's iterates are the same as in
    the single-GPU run; the per-sim reductions are batch-size independent, kernels.cu kRed*)."""
    lo, hi = shard_range(inp["B"], world, rank)
    out = dict(inp)
    for k in PER_SIM_KEYS:
        if out.get(k) is not None:
            out[k] = out[k][lo:hi]
    out["B"] = hi - lo
    out["shard"] = (lo, hi)
    if inp["cfg"].per_sim_youngs:
        out["youngs_ref"] = shared_youngs_ref(inp["youngs"], accel)
    return out


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
