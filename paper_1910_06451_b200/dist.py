"""Host-side multi-GPU plumbing for the query-sharded (weak-scaling) bench path.

Queries are independent units: every rank scores its own batch against
a replicated model, so the data path has no collective. The collectives are the model
replication after a model update (one broadcast of the packed model), the
timing barrier and the max-over-ranks reduction of the measured time.
Works with the nccl (GPU) and gloo (CPU tests) backends.
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
