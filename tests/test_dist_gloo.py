"""Multi-GPU host logic on CPU: world size 2 over gloo (127.0.0.1).

Covers what bench.py does per batch on N GPUs, with the oracle standing in
for the per-rank device compute: rank 0 produces the batch, it is broadcast
into every rank's buffers (identical replicas), each rank ingests it and
generates its walk-id shard, and the gathered shards equal one process
generating every walk id (RNG keyed by global walk id). Also checks the
max-over-ranks timing and sum-of-hops reductions."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_16182_b200.dist import all_max, all_sum, broadcast_batch, strong_shard, weak_shard

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    from oracle.py import Cfg, COracle

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    co = COracle()
    B = 4000
    buf = [torch.zeros(B, dtype=torch.int64) for _ in range(3)]
    if rank == 0:
        e = co.gen_stream(300, 0, B, 5)
        for i in range(3):
            buf[i].copy_(torch.from_numpy(np.ascontiguousarray(e[:, i])))
    broadcast_batch(buf, src=0)
    edges = np.stack([b.numpy() for b in buf], 1)
    # every rank holds the identical replica
    digest = torch.tensor([int(np.bitwise_xor.reduce(edges.ravel() * 1000003 % (1 << 61)))], dtype=torch.int64)
    allg = [torch.zeros_like(digest) for _ in range(world)]
    dist.all_gather(allg, digest)
    same = all(int(x) == int(digest) for x in allg)
    # each rank's walk shard, generated with global ids
    per_rank = 700
    lo, hi = weak_shard(rank, world, per_rank)
    cfg = Cfg(walk_length=12, start_mode=1, total_walks=per_rank * world, bias=2, seed=7)
    walks, st = co.generate(edges, 0, cfg, variant=2)
    mine = walks["nodes"].reshape(-1, walks["stride"])[lo:hi]
    hops = float(walks["lengths"][lo:hi].astype(np.int64).clip(min=1).sum() - (hi - lo))
    tot_hops = all_sum(hops)
    slowest = all_max(float(rank + 1))
    parts = [torch.zeros((per_rank, walks["stride"]), dtype=torch.int64) for _ in range(world)]
    dist.all_gather(parts, torch.from_numpy(np.ascontiguousarray(mine)))
    if rank == 0:
        union = torch.cat(parts).numpy()
        q.put((same, np.array_equal(union, walks["nodes"].reshape(-1, walks["stride"])), tot_hops,
               float(st["hops"]), slowest))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_replica_and_walk_shards():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    same, union_ok, tot_hops, full_hops, slowest = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert same, "replicas differ after broadcast"
    assert union_ok, "gathered walk shards != single-process walk set"
    assert tot_hops == full_hops
    assert slowest == 2.0


def test_shard_ranges_partition():
    for world in (1, 2, 3, 8):
        ranges = [strong_shard(r, world, 1001) for r in range(world)]
        assert ranges[0][0] == 0 and ranges[-1][1] == 1001
        assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
        w = [weak_shard(r, world, 50) for r in range(world)]
        assert w[-1][1] == 50 * world
