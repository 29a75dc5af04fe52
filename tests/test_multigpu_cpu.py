"""CPU tier (gloo, world_size 2): the N>1 path of bench.py — request-sharded replicas with no
collective on the data path; only the final metric reduction crosses ranks (max of device
time, sum of tokens). Runs on 127.0.0.1 with two processes."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = 5
    base = bench.shard_base(rank, n)
    prompts, outl = bench.prompts_for(base, n, 32000, bench.IN_RANGE, bench.OUT_RANGE)
    stats = torch.tensor([10.0 + rank, 100.0 * (rank + 1), 2.0 * (rank + 1), 7.0], dtype=torch.float64)
    agg = bench.aggregate(stats, dist)
    q.put((rank, base, [p[:8] for p in prompts], outl, agg))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_replicas_and_reduction():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # disjoint shards whose union is exactly the single-rank workload of 2n requests
    single, single_out = bench.prompts_for(0, 10, 32000, bench.IN_RANGE, bench.OUT_RANGE)
    assert out[0][1] == 0 and out[1][1] == 5
    assert out[0][2] + out[1][2] == [p[:8] for p in single]
    assert out[0][3] + out[1][3] == single_out
    # whole-job reduction: max device time / wall, summed tokens
    for _, _, _, _, agg in out:
        assert agg == [11.0, 300.0, 4.0, 14.0]


def test_single_rank_reduction_is_identity():
    stats = torch.tensor([1.5, 2.0, 3.0, 4.0], dtype=torch.float64)
    assert bench.aggregate(stats, None) == [1.5, 2.0, 3.0, 4.0]


def test_trace_shards_partition_the_arrivals():
    """Request-sharded trace replay: rank r replays trace indices r, r+N, ... (disjoint, union =
    the whole trace, arrival order kept within a shard)."""
    import bench
    trace = [(float(i), 10 + i % 5, 4) for i in range(37)]
    for world in (1, 2, 4, 8):
        shards = [bench.shard_trace(trace, r, world) for r in range(world)]
        seen = sorted(j for s in shards for j, _ in s)
        assert seen == list(range(len(trace)))
        for s in shards:
            assert [rec[0] for _, rec in s] == sorted(rec[0] for _, rec in s)


def _tp_boot(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    uid = bench.tp_bootstrap(dist, rank, lambda: bytes(range(128)))
    q.put((rank, uid))
    dist.destroy_process_group()


def test_tp_bootstrap_broadcasts_the_nccl_id():
    """Config-5 TP bring-up: every rank receives rank 0's 128-byte ncclUniqueId (gloo, world 2)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_tp_boot, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
    assert got[0] == got[1] == bytes(range(128))
