"""World-size-2 gloo test of the multi-GPU host logic (query sharding + max-over-ranks
timing), run on CPU."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch.distributed as dist

    import workloads as W
    from paper_1910_06451_b200 import dist as fd
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ws, r, lr = fd.world()
    base = W.score_workload("headline", n_queries=1000).queries
    q = fd.shard_queries(base, r)
    local_ms = 10.0 + 5.0 * r  # rank 1 is the slow one
    mx = fd.max_over_ranks(local_ms)
    # model replication: rank 0's packed model overwrites every other rank's buffer
    import torch
    model = torch.full((1000,), float(r + 1), dtype=torch.float32) if r == 0 else torch.zeros(1000)
    fd.broadcast_model(model, src=0)
    lo, hi = fd.shard_range(1001, r, ws)
    out[rank] = (ws, r, float(q[0, 0]), float(q.mean()), mx, fd.aggregate_rate(len(q), ws, mx),
                 float(model.sum()), (lo, hi))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_sharding_and_timing():
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    r0, r1 = out[0], out[1]
    assert r0[0] == r1[0] == 2 and (r0[1], r1[1]) == (0, 1)
    assert r0[2] != r1[2]  # each rank scores its own batch
    assert abs(r0[3]) < 0.2 and abs(r1[3]) < 0.2  # same U[-pi, pi] distribution
    assert r0[4] == r1[4] == 15.0  # max over ranks, seen identically everywhere
    assert r0[5] == r1[5] == pytest.approx(2 * 1000 / 15e-3)
    assert r0[6] == r1[6] == 1000.0  # the broadcast model is rank 0's everywhere
    assert r0[7] == (0, 501) and r1[7] == (501, 1001)  # contiguous shards cover the batch


def test_shard_range_partitions():
    from paper_1910_06451_b200 import dist as fd
    for n in (0, 1, 7, 1000, 1001):
        for ws in (1, 2, 3, 8):
            parts = [fd.shard_range(n, r, ws) for r in range(ws)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(parts[i][1] == parts[i + 1][0] for i in range(ws - 1))
            sizes = [hi - lo for lo, hi in parts]
            assert max(sizes) - min(sizes) <= 1


def test_single_process_defaults():
    from paper_1910_06451_b200 import dist as fd
    base = np.zeros((4, 7), np.float32)
    assert fd.shard_queries(base, 0) is base
    assert fd.max_over_ranks(3.5) == 3.5
    assert fd.aggregate_rate(10, 1, 1.0) == 10_000.0


def _strong_worker(rank, world, port, out):
    """Strong scaling: one fixed batch cut into contiguous shards, a per-unit function on
    each shard (a CPU stand-in for the per-rank fastron_query_packed / fastron_edge_check),
    results all-gathered back into batch order."""
    import torch
    import torch.distributed as dist

    import workloads as W
    from paper_1910_06451_b200 import dist as fd
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    q = torch.from_numpy(W.score_workload("headline", n_queries=1001).queries)
    seen = []

    def score_fn(qs):  # per-query: (fp32 "score", int8 "label")
        seen.append(len(qs))
        s = qs.sum(dim=1)
        return s, torch.where(s > 0, 1, -1).to(torch.int8)

    s, l = fd.sharded_map(score_fn, len(q), q)
    ew = W.edge_workload(n_edges=37, n_supports=1)
    qa, qb = torch.from_numpy(ew.qa), torch.from_numpy(ew.qb)

    def edge_fn(a, b):  # per-edge: (uint8 "in_collision", int32 "hit index")
        d = (b - a).abs().max(dim=1).values
        return (d > 3.0).to(torch.uint8), torch.where(d > 3.0, (d * 10).to(torch.int32), -1)

    hit, idx = fd.sharded_map(edge_fn, len(qa), qa, qb)
    ref_s = q.sum(dim=1)
    ref_hit = ((qb - qa).abs().max(dim=1).values > 3.0).to(torch.uint8)
    out[rank] = (seen[0], bool(torch.equal(s, ref_s)), bool(torch.equal(l, torch.where(ref_s > 0, 1, -1).to(torch.int8))),
                 bool(torch.equal(hit, ref_hit)), int(idx.shape[0]), str(hit.dtype), str(idx.dtype))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_strong_partition_gathers_in_batch_order(world):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_strong_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    from paper_1910_06451_b200 import dist as fd
    for r in range(world):
        lo, hi = fd.shard_range(1001, r, world)
        shard_n, s_ok, l_ok, hit_ok, n_idx, hd, idd = out[r]
        assert shard_n == hi - lo  # each rank scored exactly its contiguous shard
        assert s_ok and l_ok and hit_ok and n_idx == 37  # every rank holds the whole batch, in order
        assert hd == "torch.uint8" and idd == "torch.int32"
