"""The multi-GPU replica group through the C ABI (twg_group_*):
NCCL broadcast of each batch into the replica window (16-B wire format for
32-bit ids, 24-B for wider ones), the per-batch replica hash, and sharded
walk generation. The box has one GPU, so the group runs with one rank (a
real NCCL communicator of size 1: every product code path runs, the
broadcast degenerates to the root's own wire planes); the hash must equal
an independently ingested replica's, and the replica must equal the oracle's
window after every batch (replay.cpp:16-53 loop)."""
import ctypes as C

import numpy as np
import pytest

from tests.test_gpu_append import _ordered_stream
from tests.test_gpu_parity import assert_store, assert_walks, to_cfg
from oracle.py import Cfg

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def group(tw):
    ctx = tw.default_context()
    g = tw.ReplicaGroup(ctx, 1, 0, tw.group_unique_id())
    yield g
    g.close()


def _device_cols(batch):
    import torch

    b = np.ascontiguousarray(batch)
    return [torch.from_numpy(np.ascontiguousarray(b[:, k])).cuda() for k in range(3)]


@pytest.mark.parametrize("host", [False, True])
def test_group_replica_matches_oracle_every_batch(tw, co, group, host):
    import torch

    batches = _ordered_stream(3, 10, 4000, 300, 1000, skew=True)
    exp_stats, exp_dumps = co.window_run(batches, 2500, 0, every=True)
    w = tw.WindowManager(2500)
    plain = tw.WindowManager(2500)
    for b, (es, _), ed in zip(batches, exp_stats, exp_dumps):
        if host:
            gs = group.ingest(w, 0, b)
        else:
            cols = _device_cols(b)
            torch.cuda.synchronize()
            gs = group.ingest_device(w, 0, *(c.data_ptr() for c in cols), len(b))
        st = gs.local
        assert (st.ingested, st.dropped_late, st.evicted, st.retained) == (
            es["ingested"], es["dropped_late"], es["evicted"], es["retained"])
        assert gs.replicas_agree and gs.wire_bytes_per_edge == 16 and gs.edges == len(b)
        snap = w.snapshot()
        assert_store(snap, ed)
        plain.ingest_batch(b)
        # an independently ingested replica hashes the same
        assert tw.replica_hash(plain.snapshot(), len(b)) == gs.replica_hash


def test_group_wide_ids_take_24_byte_wire(tw, co, group):
    rs = np.random.default_rng(11)
    n = 3000
    t = np.sort(rs.integers(0, 5000, n))
    ids = (1 << 40) + rs.integers(0, 500, (n, 2)) * 7919
    b = np.stack([ids[:, 0], ids[:, 1], t], 1)
    w = tw.WindowManager(1 << 40)
    gs = group.ingest(w, 0, b)
    assert gs.wire_bytes_per_edge == 24 and gs.replicas_agree
    assert_store(w.snapshot(), co.build(b, 0))


def test_replica_hash_detects_a_difference(tw):
    batches = _ordered_stream(5, 4, 3000, 200, 1000)
    a, b = tw.WindowManager(10 ** 9), tw.WindowManager(10 ** 9)
    for x in batches:
        a.ingest_batch(x)
    bad = [x.copy() for x in batches]
    bad[-1][17, 1] = (bad[-1][17, 1] + 1) % 200
    for x in bad:
        b.ingest_batch(x)
    assert tw.replica_hash(a.snapshot()) != tw.replica_hash(b.snapshot())
    c = tw.WindowManager(10 ** 9)
    for x in batches:
        c.ingest_batch(x)
    assert tw.replica_hash(a.snapshot()) == tw.replica_hash(c.snapshot())


def test_group_generate_equals_generate_walks(tw, co, group):
    batches = _ordered_stream(7, 6, 5000, 400, 1000, skew=True)
    w = tw.WindowManager(3000)
    for b in batches:
        group.ingest(w, 0, b)
    snap = w.snapshot()
    for c in (Cfg(walk_length=16, start_mode=1, total_walks=3000, bias=2, start_bias=0, seed=3),
              Cfg(walk_length=12, start_mode=0, walks_per_node=3, bias=1, start_bias=0, seed=4)):
        cfg = to_cfg(tw, c)
        loc, glob = tw.WalkStats(), tw.WalkStats()
        ws = group.generate(snap, cfg, variant=tw.Variant.FullWalk, stats=loc, global_stats=glob)
        ref_ws = tw.generate_walks(snap, cfg, variant=tw.Variant.FullWalk)
        assert np.array_equal(ws.nodes, ref_ws.nodes) and np.array_equal(ws.times, ref_ws.times)
        assert loc.hops == glob.hops and loc.walks == glob.walks and glob.hops > 0


def test_group_staged_pipeline(tw, co, group):
    """stage(k+1) while k is ingested: two slots alternate, results equal the oracle's."""
    batches = _ordered_stream(9, 8, 3000, 250, 1000)
    exp_stats, exp_dumps = co.window_run(batches, 2000, 0, every=True)
    w = tw.WindowManager(2000)
    group.stage_host(0, 0, batches[0])
    for k in range(len(batches)):
        if k + 1 < len(batches):
            group.stage_host((k + 1) % 2, 0, batches[k + 1])
        gs = group.ingest_staged(w, k % 2)
        assert gs.replicas_agree and gs.local.retained == exp_stats[k][0]["retained"]
        assert_store(w.snapshot(), exp_dumps[k])


def test_group_errors(tw, group):
    with pytest.raises(ValueError):
        group.stage_host(2, 0, np.zeros((1, 3), np.int64))
    with pytest.raises(ValueError):
        group.stage_host(0, 3, np.zeros((1, 3), np.int64))
