"""GPU parity of the streaming append ingest (csrc/append.cu): time-ordered
batches over a stable node population take the shared log / node-arena
path (the snapshot reports is_streaming()); after EVERY batch the whole
dual index must equal the oracle's full rebuild of the same window
(WindowManager::ingest_batch, window_manager.cpp:14-62 +
EdgeStore::build, edge_store.cpp:27-254), including region relocation,
arena repacks, equal-time batch boundaries and hub-sized regions, and
walks on the streaming snapshots must equal the oracle's walks."""
import numpy as np
import pytest

from oracle.py import Cfg
from tests.test_gpu_parity import STORE_KEYS, assert_store, assert_walks, to_cfg

pytestmark = pytest.mark.gpu


def _ordered_stream(seed, nb, n, nodes, step, skew=False, tie_boundary=False):
    """Time-ordered batches: batch b covers times [b*step, (b+1)*step). With
    tie_boundary the first edge of every batch repeats the previous batch's
    last time with the largest ids (so the canonical concatenation still
    holds and the boundary groups/marks must merge)."""
    rs = np.random.default_rng(seed)
    out, last_t = [], None
    for b in range(nb):
        t = np.sort(b * step + rs.integers(0, step, n))
        s = rs.integers(0, nodes, n)
        if skew:
            d = np.minimum((nodes * rs.random(n) ** 3).astype(np.int64), nodes - 1)
        else:
            d = rs.integers(0, nodes, n)
        d[: n // 40] = s[: n // 40]  # self-loops
        e = np.stack([s, d, t], 1)
        e = e[np.lexsort((e[:, 1], e[:, 0], e[:, 2]))]
        if tie_boundary and last_t is not None:
            e[0] = (nodes - 1, nodes - 1, last_t)
        last_t = int(e[-1, 2])
        out.append(e)
    return out


def _run(tw, co, batches, duration, mode, check_walks=False):
    exp_stats, exp_dumps = co.window_run(batches, duration, mode, every=True)
    w = tw.WindowManager(duration, tw.DirectionMode(mode))
    streaming = 0
    for i, (b, (es, eb), ed) in enumerate(zip(batches, exp_stats, exp_dumps)):
        st = w.ingest_batch(b)
        assert (st.ingested, st.dropped_late, st.evicted, st.retained) == (
            es["ingested"], es["dropped_late"], es["evicted"], es["retained"])
        assert w.window_bounds() == eb
        snap = w.snapshot()
        streaming += snap.is_streaming()
        assert_store(snap, ed)
        if check_walks and i in (3, len(batches) - 1):
            _check_walks(tw, co, snap, ed, mode)
    return streaming


def _check_walks(tw, co, snap, ed, mode):
    edges = np.stack([ed["src_ext"], ed["dst_ext"], ed["t"]], 1)
    dirs = [0, 1] if mode == 2 else [0 if mode == 0 else 1]
    for direction in dirs:
        for bias in (0, 1, 2, 3):
            for start_mode in (0, 1):
                c = Cfg(walk_length=12, start_mode=start_mode, walks_per_node=2, total_walks=700, bias=bias,
                        start_bias=bias, direction=direction, seed=5)
                exp, _ = co.generate(edges, mode, c)
                # fresh handle each time: the weighted configurations run on
                # the snapshot's contiguous form, the others on the slices;
                # FullWalk takes the walk-record path (hop_rec) for the
                # forward index biases, Coop the ring path
                for variant in (tw.Variant.Coop, tw.Variant.FullWalk):
                    ws = tw.generate_walks(snap, to_cfg(tw, c), variant=variant)
                    assert_walks(ws, exp)
        c = Cfg(walk_length=10, start_mode=1, total_walks=500, bias=3, start_bias=0, node2vec=1, p=0.5, q=2.0,
                direction=direction, seed=9)
        exp, _ = co.generate(edges, mode, c)
        assert_walks(tw.generate_walks(snap, to_cfg(tw, c)), exp)


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_append_every_batch_bit_exact(tw, co, mode):
    """14 batches over 200 nodes: relocations every few batches, arena
    repacks; every snapshot after the first is a streaming one."""
    batches = _ordered_stream(41 + mode, 14, 3000, 200, 100)
    n = _run(tw, co, batches, 250, mode, check_walks=True)
    assert n == len(batches) - 1


@pytest.mark.parametrize("mode,step", [(2, 200000), (0, 1 << 33)])
def test_append_two_pass_sort_and_time_span(tw, co, mode, step):
    """70K nodes (bucket sort over two 8-bit digit passes, the owner-digit
    histogram fused into the statistics pass), 600K-edge batches (every node
    present: the fast route; interior statistics tiles staged by TMA bulk
    copies), and either a batch time span
    below 2^32 (12-B sort payloads) or of 2^33 (16-B payloads: the time does
    not fit a u32 offset): the index after every batch and the walks on the
    last snapshot equal the oracle's."""
    batches = _ordered_stream(90 + mode, 4, 600000, 70000, step)
    n = _run(tw, co, batches, 2 * step, mode, check_walks=step < (1 << 32))
    assert n == len(batches) - 1


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_append_shuffled_ties_across_sort_tiles(tw, co, mode):
    """Time-ordered batches whose equal-time runs (about 6 edges, up to ~25)
    arrive in random order: the statistics pass writes them to the log in
    canonical (src, dst) order, so around every 1536-edge tile boundary a run
    straddles, the input order (the statistics pass's per-tile owner-digit
    counts) and the canonical order (the first bucket-sort pass's items)
    disagree — the first pass's precomputed tile offsets must be corrected for
    exactly that run (OwnerIn::run_fix). 70K nodes (two digit passes),
    600K-edge batches on the fast route; the index after every batch and the
    walks on the last snapshot equal the oracle's."""
    rs = np.random.default_rng(77 + mode)
    batches = []
    for b in range(4):
        n, nodes, step = 600000, 70000, 100000
        t = np.sort(b * step + rs.integers(0, step, n))
        s = rs.integers(0, nodes, n)
        d = np.minimum((nodes * rs.random(n) ** 2).astype(np.int64), nodes - 1)
        e = np.stack([s, d, t], 1)
        batches.append(e[np.lexsort((rs.random(n), e[:, 2]))])  # time order, runs shuffled
    n = _run(tw, co, batches, 2 * 100000, mode, check_walks=mode != 2)
    assert n == len(batches) - 1


@pytest.mark.parametrize("mode", [0, 2])
def test_append_arena_exhausted_mid_stream(tw, co, mode, monkeypatch):
    """The plan, the relocation copies and the placement are queued back to
    back and the plan's scalars read once at the end; when the plan finds the
    node arena exhausted, the queued kernels must do nothing and the host must
    repack into a fresh arena. TWG_ARENA_TIGHT sizes every fresh arena at the
    minimum a repack needs, so streaming batches keep exhausting it: several
    repacks happen, and the index after every batch (and the walks) still
    equals the oracle's."""
    monkeypatch.setenv("TWG_ARENA_TIGHT", "1")
    batches = _ordered_stream(61 + mode, 12, 3000, 150, 100, skew=True)
    exp_stats, exp_dumps = co.window_run(batches, 300, mode, every=True)
    w = tw.WindowManager(300, tw.DirectionMode(mode))
    serials = []
    for i, (b, ed) in enumerate(zip(batches, exp_dumps)):
        w.ingest_batch(b)
        snap = w.snapshot()
        assert_store(snap, ed)
        if snap.is_streaming():
            serials.append(snap.layout()["arena_serial"])
        if i == len(batches) - 1:
            _check_walks(tw, co, snap, ed, mode)
    assert len(serials) == len(batches) - 1
    assert len(set(serials)) >= 3, serials  # repacks after the first streaming batch


@pytest.mark.parametrize("mode", [0, 2])
def test_append_tie_boundary(tw, co, mode):
    """Batch boundaries sharing a timestamp: the first batch group and the
    first batch mark of a node merge with the survivors' last ones."""
    batches = _ordered_stream(7, 10, 2000, 150, 60, tie_boundary=True)
    # walks too: a merged boundary group's record (the sampled-start line) is rebuilt
    n = _run(tw, co, batches, 150, mode, check_walks=True)
    assert n == len(batches) - 1


@pytest.mark.parametrize("mode", [1, 2])
def test_append_hub_regions(tw, co, mode):
    """Skewed destinations (dst = N*u^3): the hub regions exceed the big-copy
    threshold (2048 live entries), so relocations use the CTA-grid copy."""
    batches = _ordered_stream(3, 8, 20000, 300, 1000, skew=True)
    n = _run(tw, co, batches, 2500, mode)
    assert n == len(batches) - 1


def test_append_population_change_falls_back(tw, co):
    """A node leaving the window (or a new one arriving) changes the dense
    ids: that batch takes the rewrite route from the streaming snapshot's
    contiguous form, the following ones resume appending."""
    batches = _ordered_stream(5, 8, 2000, 100, 50)
    # batch 4 introduces a brand-new node 1000
    batches[4] = batches[4].copy()
    batches[4][-1] = (1000, 3, batches[4][-1, 2])
    exp_stats, exp_dumps = co.window_run(batches, 120, 0, every=True)
    w = tw.WindowManager(120)
    kinds = []
    for b, ed in zip(batches, exp_dumps):
        w.ingest_batch(b)
        kinds.append(w.snapshot().is_streaming())
        assert_store(w.snapshot(), ed)
    assert kinds[4] is False and kinds[3] is True


def test_append_held_snapshots_stay_valid(tw, co):
    """The retired snapshot stays readable while the next batches append."""
    batches = _ordered_stream(13, 6, 2000, 100, 50)
    exp_stats, exp_dumps = co.window_run(batches, 120, 0, every=True)
    w = tw.WindowManager(120)
    snaps = []
    for b in batches:
        w.ingest_batch(b)
        snaps.append(w.snapshot())
    # every held snapshot (not only the current one) still reads back exactly
    for s, ed in zip(snaps, exp_dumps):
        assert_store(s, ed, keys=["src_ext", "dst_ext", "t", "ts_off", "n_off", "mk_time", "mk_start", "ref_edge"])


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_append_node_leaves_window(tw, co, mode):
    """Node 7 stops appearing after batch 2: once its last edge is evicted the
    fast route's population check aborts (nothing published) and the general
    route re-densifies the ids; bit-exact after every batch."""
    batches = _ordered_stream(19, 9, 2000, 100, 50)
    for b in range(3, 9):
        e = batches[b].copy()
        e[e[:, 0] == 7, 0] = 8
        e[e[:, 1] == 7, 1] = 9
        batches[b] = e[np.lexsort((e[:, 1], e[:, 0], e[:, 2]))]
    exp_stats, exp_dumps = co.window_run(batches, 120, mode, every=True)
    w = tw.WindowManager(120, tw.DirectionMode(mode))
    counts = []
    for b, (es, eb), ed in zip(batches, exp_stats, exp_dumps):
        st = w.ingest_batch(b)
        assert (st.evicted, st.retained) == (es["evicted"], es["retained"])
        counts.append(w.snapshot().node_count())
        assert_store(w.snapshot(), ed)
    assert counts[0] == 100 and counts[-1] == 99


def test_c5_law_stream_small_scale(tw, co):
    """The bench's own pipeline at 1/1000 scale: the C5 stream law generated
    on the device (twg_synth_stream_device), ingested batch by batch through
    the device-resident fast route, every snapshot compared with the oracle's
    window over the same (host-generated) stream, and exp-index walks on the
    last one compared with the oracle's."""
    import torch
    from bench import Workload
    from oracle.py import Cfg
    wl = Workload(0.001)
    B, lib = wl.batch_edges, tw._abi.load()
    ctx = tw.Context(0)
    w = tw.WindowManager(wl.window, weights=False, adjacency=False, ctx=ctx)
    dev = [torch.empty(B, dtype=torch.int64, device="cuda") for _ in range(3)]
    batches = [co.gen_stream(wl.nodes, b * B, B, wl.seed) for b in range(wl.prefill + 5)]
    exp_stats, exp_dumps = co.window_run(batches, wl.window, 0, every=True)
    streaming = 0
    for b, ed in enumerate(exp_dumps):
        assert lib.twg_synth_stream_device(ctx.handle, wl.nodes, b * B, B, wl.seed, dev[0].data_ptr(),
                                           dev[1].data_ptr(), dev[2].data_ptr()) == 0
        w.ingest_batch_device(dev[0].data_ptr(), dev[1].data_ptr(), dev[2].data_ptr(), B, stats=False)
        snap = w.snapshot()
        streaming += snap.is_streaming()
        assert_store(snap, ed, keys=["src_ext", "dst_ext", "t", "ts_off", "ts_time", "n_off", "n_tsidx", "mk_time",
                                     "mk_start", "ref_edge", "ref_nbr", "ext"])
    assert streaming >= 3
    edges = np.stack([exp_dumps[-1]["src_ext"], exp_dumps[-1]["dst_ext"], exp_dumps[-1]["t"]], 1)
    for bias, start_bias in ((2, 0), (3, 3), (3, 0)):  # exp-index; exp-weight (the reference default) both ways
        c = Cfg(walk_length=wl.walk_length, start_mode=1, total_walks=5000, bias=bias, start_bias=start_bias,
                seed=wl.seed)
        exp, _ = co.generate(edges, 0, c)
        snap = w.snapshot()
        assert snap.is_streaming()
        assert_walks(tw.generate_walks(snap, to_cfg(tw, c), variant=tw.Variant.FullWalk), exp)


@pytest.mark.parametrize("mode", [0, 2])
def test_append_ring_rebase(tw, co, mode, monkeypatch):
    """Ring positions are u32 and rebased only when a ring moves; a ring whose
    logical end would pass the rebase bound (2^31 by default, lowered to 64
    here through TWG_RING_REBASE) is relocated to logical 0 although it
    still fits. With the bound this low nearly every ring is rebased every
    batch; the whole index must stay bit-exact after every batch."""
    monkeypatch.setenv("TWG_RING_REBASE", "64")
    batches = _ordered_stream(57 + mode, 10, 3000, 60, 100)
    n = _run(tw, co, batches, 350, mode, check_walks=True)
    assert n == len(batches) - 1
