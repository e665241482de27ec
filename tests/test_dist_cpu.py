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
    out[rank] = (ws, r, float(q[0, 0]), float(q.mean()), mx, fd.aggregate_rate(len(q), ws, mx))
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


def test_single_process_defaults():
    from paper_1910_06451_b200 import dist as fd
    base = np.zeros((4, 7), np.float32)
    assert fd.shard_queries(base, 0) is base
    assert fd.max_over_ranks(3.5) == 3.5
    assert fd.aggregate_rate(10, 1, 1.0) == 10_000.0
