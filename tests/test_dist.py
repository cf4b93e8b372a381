"""Multi-process (world_size 2 and 3, gloo, CPU) coverage of bench.py's N > 1 plumbing
(SURVEY.md §8(e), strong scaling of one fixed batch): contiguous shard ranges, max-over-ranks
timing, whole-job aggregation, the broadcast of rank 0's IPC handles, and the fallback gather
of the ranks' shards into rank 0's buffers."""
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
    P = 10
    # every rank draws the SAME batch (one fixed batch, strong scaling) and owns a shard of it
    _, X = config_system("tiny", seed=1, points=P)
    t = torch.from_numpy(X).reshape(-1)
    gathered = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(gathered, t)
    same = all(torch.equal(gathered[0], g) for g in gathered[1:])
    local_ms = 10.0 + 5.0 * rank  # the last rank is the slow one
    ms = bench.max_over_ranks(local_ms, world)
    val = bench.aggregate_value(P, 4, ms)
    # rank 0's "IPC handles" (opaque bytes + offsets) reach every rank unchanged
    payload = [(bytes(range(64)), 0), (bytes(range(64, 128)), 4096)] if rank == 0 else None
    got = bench.share_handles(rank, world, payload)
    # fallback gather: rank r fills its shard rows with r + 1, rank 0 ends up with all of them
    full = torch.zeros((P, 3), dtype=torch.float64)
    a, b = bench.shard_range(rank, world, P)
    full[a:b] = rank + 1
    bench.gather_to_rank0(rank, world, full, lambda r: bench.shard_range(r, world, P))
    out[rank] = (ms, val, same, got, full.numpy().copy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_multi_rank_gloo_plumbing(world):
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    slow = 10.0 + 5.0 * (world - 1)
    for r in range(world):
        ms, val, same, got, _ = out[r]
        assert ms == slow  # max over ranks
        assert val == pytest.approx(10 * 4 / (slow * 1e-3))  # the batch's points, not per rank
        assert same
        assert got == [(bytes(range(64)), 0), (bytes(range(64, 128)), 4096)]
    full0 = out[0][4]
    import bench
    for r in range(world):
        a, b = bench.shard_range(r, world, 10)
        assert (full0[a:b] == r + 1).all()


def test_shard_ranges_cover_points():
    """The sharding rule (include/phc.h): contiguous equal ranges [g P / G, (g+1) P / G) cover
    every point exactly once, in order."""
    import bench
    for P in (0, 1, 7, 4096, 65536, 4097):
        for G in (1, 2, 3, 4, 8):
            r = [bench.shard_range(g, G, P) for g in range(G)]
            assert r[0][0] == 0 and r[-1][1] == P
            assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
            assert max(b - a for a, b in r) - min(b - a for a, b in r) <= 1


def test_nominal_peak_and_parse_defaults():
    """The roofline denominator is derived from unit counts and the clock, and the
    default workload is the largest single-GPU config (configs[4] as its 4,096-point batch)."""
    import bench
    assert bench.nominal_fp64_tflops() == pytest.approx(148 * 64 * 2 * 1.965e9 / 1e12)
    a = bench.parse([])
    assert a.workload == "large_batch" and a.gpus == 1 and a.warmup >= 3
    assert np.isclose(bench.aggregate_value(4096, 10, 1000.0), 40960.0)
