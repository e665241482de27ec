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
