"""Multi-process (world_size 2, gloo, CPU) coverage of the N>1 bench plumbing: per-rank
seeds (weak scaling: disjoint batches), max-over-ranks timing, whole-job aggregation, and
that the ranks' synthetic batches differ while each is reproducible."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from synthetic import config_system
    seed = bench.rank_seed(rank)
    _, X = config_system("tiny", seed=seed, points=3)
    # gather every rank's points to check they differ (weak scaling: disjoint work)
    t = torch.from_numpy(X).reshape(-1)
    gathered = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(gathered, t)
    local_ms = 10.0 + 5.0 * rank  # rank 1 is the slow one
    ms = bench.max_over_ranks(local_ms, world)
    val = bench.aggregate_value(world, 65536, 4, ms)
    out[rank] = (seed, ms, val, all(not torch.equal(gathered[0], g) for g in gathered[1:]))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_aggregation():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    assert out[0][0] != out[1][0]
    assert out[0][1] == out[1][1] == 15.0  # max over ranks
    assert out[0][2] == pytest.approx(2 * 65536 * 4 / 15e-3)
    assert out[0][3] and out[1][3]


def test_shard_ranges_cover_points():
    """The batch call's sharding rule (include/phc.h): contiguous equal ranges
    [g P / G, (g+1) P / G) cover every point exactly once, in order."""
    for P in (0, 1, 7, 65536, 4097):
        for G in (1, 2, 3, 4, 8):
            r = [(g * P // G, (g + 1) * P // G) for g in range(G)]
            assert r[0][0] == 0 and r[-1][1] == P
            assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
            assert max(b - a for a, b in r) - min(b - a for a, b in r) <= 1
