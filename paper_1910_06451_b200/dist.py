"""Host-side multi-GPU plumbing: query and edge sharding over ranks.

Queries and edges are independent units: every rank scores its units
against a replicated model, so the data path has no collective. Two partitions:
  * weak scaling (bench default): every rank its own batch of the workload's size;
  * strong scaling (bench --strong, edge checks): one fixed batch cut into contiguous
    shards (shard_range), results reassembled in batch order by gather_shards when one
    rank needs them all (an all-gather of 4-byte scores / 1-byte edge flags).
The collectives are the model replication after a model update (one broadcast of the
packed model), the timing barrier and the max-over-ranks reduction of the measured time
(DESIGN.md §8). Works with the nccl (GPU) and gloo (CPU tests) backends.
"""
from __future__ import annotations

import os

import numpy as np


def world():
    """(world_size, rank, local_rank) from the torchrun environment (1, 0, 0 when absent)."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard_queries(base_queries: np.ndarray, rank: int, seed: int = 1000) -> np.ndarray:
    """Rank 0 keeps the workload's seeded batch; rank r > 0 draws its own batch of the same
    shape and distribution (U[-pi, pi]^D) from default_rng(seed + r)."""
    if rank == 0:
        return base_queries
    rng = np.random.default_rng(seed + rank)
    return rng.uniform(-np.pi, np.pi, size=base_queries.shape).astype(np.float32)


def shard_range(n: int, rank: int, world_size: int) -> tuple:
    """Contiguous partition of n independent units (queries or edges) over the ranks, for a
    fixed total batch (strong scaling): rank r gets [lo, hi); sizes differ by at most 1."""
    base, extra = divmod(int(n), int(world_size))
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def shard(x, rank: int, world_size: int):
    """Rank `rank`'s contiguous shard of the rows of x (shard_range), a view."""
    lo, hi = shard_range(len(x), rank, world_size)
    return x[lo:hi]


def _initialised():
    import torch.distributed as dist
    return dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1


def gather_shards(local, n_total: int):
    """All-gather the ranks' contiguous shards (shard_range order) of a batch of n_total
    rows into the whole batch, on every rank (shards are padded to the largest size for
    the collective and cut back). `local` is a torch tensor on the backend's device."""
    import torch
    import torch.distributed as dist
    if not _initialised():
        return local
    ws = dist.get_world_size()
    sizes = [shard_range(n_total, r, ws) for r in range(ws)]
    m = max(hi - lo for lo, hi in sizes)
    buf = torch.zeros((m,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    buf[:local.shape[0]] = local
    parts = [torch.empty_like(buf) for _ in range(ws)]
    dist.all_gather(parts, buf)
    return torch.cat([parts[r][:hi - lo] for r, (lo, hi) in enumerate(sizes)], dim=0)


def sharded_map(fn, n_total: int, *arrays, gather: bool = True):
    """Strong-scaling driver for independent units: this rank applies fn to its contiguous
    shard of every array (rows), e.g. fn = a fastron_edge_check of the shard's edges or a
    fastron_query_packed of the shard's configurations; the per-unit outputs (a tensor or a
    tuple of tensors) are all-gathered back into batch order when `gather`."""
    import torch.distributed as dist
    ws, rank = (dist.get_world_size(), dist.get_rank()) if _initialised() else (1, 0)
    out = fn(*[shard(a, rank, ws) for a in arrays])
    if not gather:
        return out
    if isinstance(out, tuple):
        return tuple(None if o is None else gather_shards(o, n_total) for o in out)
    return gather_shards(out, n_total)


def broadcast_model(packed, src: int = 0):
    """Replicate a packed model (fastron_model_pack output, a flat tensor) from rank `src`
    to every rank in place — one broadcast per model update (no-op on a single process)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.broadcast(packed, src=src)
    return packed


def max_over_ranks(value: float, device=None) -> float:
    """All-reduce MAX of a per-rank scalar (a no-op without an initialised process group)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def aggregate_rate(units_per_rank: int, world_size: int, max_ms: float) -> float:
    """Whole-job throughput: all ranks' units divided by the slowest rank's time."""
    return world_size * units_per_rank / (max_ms * 1e-3)
