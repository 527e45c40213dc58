"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on
the same seeded inputs. Bit-exact for every integer/index array and every
fp64 weight prefix; walks byte-identical (splitmix vs the reference RNG,
Philox vs the Philox oracle)."""
import numpy as np
import pytest

from oracle.py import Cfg

pytestmark = pytest.mark.gpu

STORE_KEYS = ["src_ext", "dst_ext", "t", "src", "dst", "ts_off", "ts_time", "ts_w", "n_off", "n_tsidx",
              "mk_time", "mk_start", "ref_edge", "wprefix", "ext", "ref_nbr", "adj_off", "adj"]


def assert_store(tw_store, oracle_dump, keys=STORE_KEYS):
    got = tw_store.dump(keys)
    for k in keys:
        exp = oracle_dump[k]
        g = got[k]
        assert g.shape == exp.shape, (k, g.shape, exp.shape)
        if g.dtype.kind == "f":
            assert np.array_equal(g.view(np.uint64), exp.astype(np.float64).view(np.uint64)), k
        else:
            assert np.array_equal(g.astype(np.int64), exp.astype(np.int64)), k


def to_cfg(tw, c: Cfg):
    return tw.WalkConfig(walk_length=c.walk_length, start_mode=tw.StartMode(c.start_mode),
                         walks_per_node=c.walks_per_node, total_walks=c.total_walks, bias=tw.BiasKind(c.bias),
                         start_bias=tw.BiasKind(c.start_bias),
                         node2vec=tw.Node2VecParams(c.p, c.q) if c.node2vec else None,
                         node2vec_temporal_adjacency=c.temporal_adjacency, direction=tw.WalkDirection(c.direction),
                         seed=c.seed, rng=tw.RngKind(c.rng))


def assert_walks(ws, exp):
    assert ws.stride == exp["stride"] and ws.walk_count == exp["walk_count"]
    assert np.array_equal(ws.lengths, exp["lengths"])
    assert np.array_equal(ws.nodes, exp["nodes"])
    assert np.array_equal(ws.times, exp["times"])


@pytest.fixture(scope="module")
def graphs(co):
    return {
        "uniform": co.gen_uniform(100, 3000, 50, 17),
        "hub": co.gen_hub_skewed(2000, 20000, 0),
        "mega": co.gen_mega_hub(1700, 23),
        "ladder": co.gen_time_ladder(20000, 256, 17),
        "ties": co.gen_uniform(20, 500, 5, 77),
        "c1": co.gen_uniform(100000, 1000000, 1000000, 1),
    }


# ------------------------------------------------------------------ index

@pytest.mark.parametrize("mode", [0, 1, 2])
@pytest.mark.parametrize("name", ["uniform", "hub", "ladder", "ties", "mega"])
def test_store_parity(tw, co, graphs, name, mode):
    assert_store(tw.EdgeStore.build(graphs[name], tw.DirectionMode(mode)), co.build(graphs[name], mode))


def test_store_c1_full(tw, co, graphs):
    """C1 (1M edges, 100K nodes): every array bit-exact."""
    assert_store(tw.EdgeStore.build(graphs["c1"], tw.DirectionMode.DirectedForward), co.build(graphs["c1"], 0))


def test_store_sparse_ids(tw, co):
    """64-bit ids force the sort-unique densify path."""
    rs = np.random.default_rng(1)
    ids = rs.integers(0, 2**62, 500)
    e = np.stack([ids[rs.integers(0, 500, 5000)], ids[rs.integers(0, 500, 5000)], rs.integers(0, 300, 5000)], 1)
    for mode in (0, 2):
        assert_store(tw.EdgeStore.build(e, tw.DirectionMode(mode)), co.build(e, mode))


def test_store_wide_keys(tw, co):
    """time span + ids too wide for one 64-bit key: two-pass canonical sort."""
    rs = np.random.default_rng(2)
    n = 20000
    e = np.stack([rs.integers(0, 3_000_000, n), rs.integers(0, 3_000_000, n), rs.integers(0, 2**40, n)], 1)
    assert_store(tw.EdgeStore.build(e, tw.DirectionMode.DirectedForward), co.build(e, 0))


def test_store_edge_cases(tw, co):
    big = (1 << 62) + 12345
    for edges in ([], [(7, 8, 3)], [(1, 1, 3), (1, 2, 3), (1, 2, 3)], [(big, big - 7, 1), (big - 7, big, 2)],
                  [(1, 2, 5), (1, 3, 5), (1, 4, 9)]):
        for mode in (0, 1, 2):
            assert_store(tw.EdgeStore.build(edges, tw.DirectionMode(mode)), co.build(edges, mode))


def test_store_rejects_negative(tw):
    with pytest.raises(ValueError):
        tw.EdgeStore.build([(1, 2, -3)])
    with pytest.raises(ValueError):
        tw.EdgeStore.build([(-1, 2, 3)])


def test_store_permutation_determinism(tw, graphs):
    e = graphs["ties"]
    a = tw.EdgeStore.build(e).dump()
    b = tw.EdgeStore.build(e[np.random.default_rng(99).permutation(len(e))]).dump()
    for k in a:
        assert np.array_equal(a[k], b[k]), k


def test_known_answer_groups(tw):
    """test_edge_store.cpp:41-58."""
    s = tw.EdgeStore.build([(1, 2, 5), (1, 3, 5), (1, 4, 9)])
    assert s.ts_group_count() == 2
    assert s.edge_slice_for_ts_group(0) == (0, 2)
    assert s.edge_slice_for_ts_group(1) == (2, 3)
    assert (s.ts_group_time(0), s.ts_group_time(1)) == (5, 9)
    a = s.find_node(1)
    lo, hi = s.node_region(a)
    assert hi - lo == 3 and s.timestamp_group_count(1) == 2
    with pytest.raises(IndexError):
        s.edge_slice_for_ts_group(2)


def test_neighborhood_queries(tw, co, graphs):
    """Γ_t(v) for all three modes vs the oracle (test_edge_store.cpp:119-134)."""
    for mode in (0, 1, 2):
        e = graphs["uniform"]
        s = tw.EdgeStore.build(e, tw.DirectionMode(mode))
        d = 1 if mode == 1 else 0
        qs = [(v, t) for v in range(0, 101, 3) for t in (0, 1, 7, 25, 49, 50)]
        got = s.temporal_neighborhoods([q[0] for q in qs], [q[1] for q in qs], tw.WalkDirection(d))
        exp = co.neighborhood(e, mode, qs, d)
        assert [tuple(int(x) for x in r) for r in got] == exp
    s = tw.EdgeStore.build([(1, 2, 2), (3, 2, 5), (4, 2, 9)], tw.DirectionMode.DirectedBackward)
    with pytest.raises(ValueError):
        s.temporal_neighborhood(2, 6, tw.WalkDirection.Forward)
    # an unknown node answers {} before the direction check (edge_store.cpp:270-282)
    r = s.temporal_neighborhood(99, 6, tw.WalkDirection.Forward)
    assert (r.start, r.end, r.group_count) == (0, 0, 0)


def test_adjacency_predicate(tw):
    """test_edge_store.cpp:215-230."""
    s = tw.EdgeStore.build([(1, 2, 1), (2, 3, 2)])
    n1, n2, n3 = s.find_node(1), s.find_node(2), s.find_node(3)
    assert s.adjacent(n1, n2) and not s.adjacent(n2, n1) and s.adjacent(n2, n3) and not s.adjacent(n1, n3)
    assert s.adjacent_after(n1, n2, 0, tw.WalkDirection.Forward)
    assert not s.adjacent_after(n1, n2, 1, tw.WalkDirection.Forward)
    u = tw.EdgeStore.build([(1, 2, 1), (2, 3, 2)], tw.DirectionMode.Undirected)
    assert u.adjacent(u.find_node(2), u.find_node(1))


# ------------------------------------------------------------------ window

def test_window_known_answers(tw):
    """test_window.cpp:25-38, :50-60, :87-103."""
    def at(times):
        return [(2 * i + 1, 2 * i + 2, t) for i, t in enumerate(times)]
    w = tw.WindowManager(10)
    w.ingest_batch(at([16, 18, 22, 25]))
    st = w.ingest_batch(at([18, 26, 30]))
    assert w.t_high() == 30 and w.window_bounds() == (20, 30)
    assert (st.ingested, st.dropped_late, st.evicted, st.retained) == (3, 1, 2, 4)
    w2 = tw.WindowManager(10)
    st = w2.ingest_batch([(t, t + 1000, t) for t in range(1, 101)])
    assert st.retained == 11 and w2.window_bounds() == (90, 100)
    w3 = tw.WindowManager(5)
    w3.ingest_batch(at([20, 22, 25]))
    st = w3.ingest_batch(at([1, 2, 3]))
    assert st.dropped_late == 3 and st.retained == 3 and w3.t_high() == 25
    with pytest.raises(tw.LogicError):
        tw.WindowManager(10).window_bounds()
    with pytest.raises(ValueError):
        tw.WindowManager(0)


def test_window_empty_batch_and_immutability(tw):
    w = tw.WindowManager(10)
    w.ingest_batch([(1, 2, 5), (3, 4, 7)])
    old = w.snapshot()
    w.ingest_batch([])
    assert w.batch_count() == 2 and w.t_high() == 7
    w.ingest_batch([(5, 6, 50), (7, 8, 60)])
    assert old.edge_count() == 2 and old.edge_at(0)[2] == 5
    assert w.snapshot().edge_count() == 2


@pytest.mark.parametrize("mode", [0, 2])
def test_window_sequence_parity(tw, co, mode):
    """Post-eviction state bit-exact after every batch (stats + final arrays)."""
    rs = np.random.default_rng(3)
    batches, base = [], 0
    for b in range(15):
        n = 2000
        t = base + rs.integers(0, 400, n)
        batches.append(np.stack([rs.integers(0, 300, n), rs.integers(0, 300, n), t], 1))
        base += 250
    batches.insert(7, np.zeros((0, 3), np.int64))
    exp_stats, exp_dump = co.window_run(batches, 500, mode)
    w = tw.WindowManager(500, tw.DirectionMode(mode))
    for b, (es, eb) in zip(batches, exp_stats):
        st = w.ingest_batch(b)
        assert (st.ingested, st.dropped_late, st.evicted, st.retained) == (
            es["ingested"], es["dropped_late"], es["evicted"], es["retained"])
        assert w.window_bounds() == eb
    assert_store(w.snapshot(), exp_dump)


def _stream_batches(seed, nb, n, nodes, span, step, ids=None, dup=True):
    """Random batches with late edges, duplicates and self-loops."""
    rs = np.random.default_rng(seed)
    out, base = [], 0
    for b in range(nb):
        t = base + rs.integers(0, span, n)
        s = rs.integers(0, nodes, n)
        d = rs.integers(0, nodes, n)
        d[: n // 50] = s[: n // 50]  # self-loops
        e = np.stack([s, d, t], 1)
        if dup:
            e[n // 2: n // 2 + n // 20] = e[: n // 20]  # exact duplicates
        if ids is not None:
            e[:, 0] = ids[e[:, 0]]
            e[:, 1] = ids[e[:, 1]]
        out.append(e)
        base += step
    return out


@pytest.mark.parametrize("mode", [0, 1, 2])
@pytest.mark.parametrize("sparse", [False, True])
def test_window_every_batch_bit_exact(tw, co, mode, sparse):
    """Streaming merge path (dense ids) and full-rebuild path (sparse 62-bit
    ids): the whole dual index after EVERY batch equals the oracle's."""
    ids = np.random.default_rng(9).integers(0, 2**62, 400) if sparse else None
    batches = _stream_batches(11 + mode, 12, 3000, 400, 300, 120, ids)
    batches.insert(4, np.zeros((0, 3), np.int64))
    exp_stats, exp_dumps = co.window_run(batches, 500, mode, every=True)
    w = tw.WindowManager(500, tw.DirectionMode(mode))
    for b, (es, eb), ed in zip(batches, exp_stats, exp_dumps):
        st = w.ingest_batch(b)
        assert (st.ingested, st.dropped_late, st.evicted, st.retained) == (
            es["ingested"], es["dropped_late"], es["evicted"], es["retained"])
        assert w.window_bounds() == eb
        assert_store(w.snapshot(), ed)


@pytest.mark.parametrize("span", [3000, 40])
def test_window_time_ordered_batches(tw, co, span):
    """Time-ordered batches take the in-register segment sort (short
    equal-time runs, span 3000) or fall back to the radix sort (runs > 32,
    span 40); both bit-exact after every batch."""
    batches = []
    for e in _stream_batches(21, 8, 2000, 300, span, span // 2):
        batches.append(e[np.argsort(e[:, 2], kind="stable")])
    for mode in (0, 1, 2):
        exp_stats, exp_dumps = co.window_run(batches, span * 2, mode, every=True)
        w = tw.WindowManager(span * 2, tw.DirectionMode(mode))
        for b, ed in zip(batches, exp_dumps):
            w.ingest_batch(b)
            assert_store(w.snapshot(), ed)


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_window_stable_node_set(tw, co, mode):
    """Fixed small population: every batch after the first keeps the node set
    (identity id remap fast path); bit-exact after every batch."""
    batches = _stream_batches(31, 8, 3000, 20, 200, 100)
    exp_stats, exp_dumps = co.window_run(batches, 300, mode, every=True)
    w = tw.WindowManager(300, tw.DirectionMode(mode))
    for b, ed in zip(batches, exp_dumps):
        w.ingest_batch(b)
        assert w.snapshot().node_count() == 20
        assert_store(w.snapshot(), ed)


def test_window_c2_replay_state(tw, co):
    """C2 shape: C1 edges sorted by time, 10 batches, Δ = span/3; every
    post-eviction snapshot bit-exact (weights included: exp-weight default)."""
    g = co.gen_uniform(100000, 1000000, 1000000, 1)
    g = g[np.argsort(g[:, 2], kind="stable")]
    bounds = tw.split_batches(g[:, 2], 100000)
    batches = [g[a:b] for a, b in bounds]
    assert len(batches) == 10
    exp_stats, exp_dumps = co.window_run(batches, 333333, 0, every=True)
    w = tw.WindowManager(333333)
    for b, ed in zip(batches, exp_dumps):
        w.ingest_batch(b)
        assert_store(w.snapshot(), ed)


def test_window_rejects_negative_admitted_id(tw):
    w = tw.WindowManager(10)
    w.ingest_batch([(1, 2, 5)])
    with pytest.raises(ValueError):
        w.ingest_batch([(-1, 2, 6)])
    assert w.batch_count() == 1 and w.snapshot().edge_count() == 1
    st = w.ingest_batch([(-1, 2, -7), (3, 4, 8)])  # negative edge is late: dropped, not an error
    assert st.dropped_late == 1 and st.retained == 2


# ------------------------------------------------------------------ walks

@pytest.mark.parametrize("mode,direction", [(0, 0), (1, 1), (2, 0), (2, 1)])
@pytest.mark.parametrize("bias", [0, 1, 2, 3])
@pytest.mark.parametrize("start_mode", [0, 1])
def test_walks_bit_exact(tw, co, graphs, mode, direction, bias, start_mode):
    cfg = Cfg(walk_length=12, start_mode=start_mode, walks_per_node=3, total_walks=3000, bias=bias,
              start_bias=(bias + 1) % 4, seed=99, direction=direction)
    g = graphs["hub"]
    exp, es = co.generate(g, mode, cfg, variant=0)
    store = tw.EdgeStore.build(g, tw.DirectionMode(mode))
    for variant in (tw.Variant.Coop, tw.Variant.CoopDirect, tw.Variant.FullWalk):
        st = tw.WalkStats()
        ws = tw.generate_walks(store, to_cfg(tw, cfg), variant=variant, stats=st)
        assert_walks(ws, exp)
        assert (st.walks, st.hops) == (es["walks"], es["hops"])
        assert st.ambiguous_draws == 0
        if variant != tw.Variant.FullWalk:
            assert st.steps == es["steps"]


def test_mega_hub_neutrality_and_tiers(tw, co, graphs):
    g = graphs["mega"]
    cfg = Cfg(walk_length=8, seed=5)
    exp, es = co.generate(g, 0, cfg)
    store = tw.EdgeStore.build(g)
    st = tw.WalkStats()
    ws = tw.generate_walks(store, to_cfg(tw, cfg), stats=st)
    assert_walks(ws, exp)
    assert st.tiers.multi_block == es["multi_block"] >= 3


def test_tier_counts_c3b(tw, graphs):
    """acceptance.cpp:276-294, golden solo=19 wc=6230 wd=4 bc=11 bd=1 mb=7 (test_output.txt:38)."""
    store = tw.EdgeStore.build(graphs["hub"])
    st = tw.WalkStats()
    tw.generate_walks(store, tw.WalkConfig(), stats=st)
    t = st.tiers
    assert (t.solo, t.warp_cached, t.warp_direct, t.block_cached, t.block_direct, t.multi_block) == \
        (19, 6230, 4, 11, 1, 7)


@pytest.mark.parametrize("temporal", [False, True])
@pytest.mark.parametrize("mode", [0, 2])
def test_node2vec_bit_exact(tw, co, graphs, temporal, mode):
    cfg = Cfg(walk_length=10, start_mode=1, total_walks=4000, bias=3, node2vec=True, p=0.5, q=2.0,
              temporal_adjacency=temporal, seed=7)
    exp, _ = co.generate(graphs["uniform"], mode, cfg)
    store = tw.EdgeStore.build(graphs["uniform"], tw.DirectionMode(mode))
    for variant in (tw.Variant.Coop, tw.Variant.FullWalk):
        assert_walks(tw.generate_walks(store, to_cfg(tw, cfg), variant=variant), exp)


@pytest.mark.parametrize("bias", [0, 1, 2, 3])
def test_philox_walks(tw, co, graphs, bias):
    cfg = Cfg(walk_length=16, start_mode=1, total_walks=3000, bias=bias, seed=5, rng=1)
    exp, _ = co.generate(graphs["hub"], 0, cfg)
    store = tw.EdgeStore.build(graphs["hub"])
    assert_walks(tw.generate_walks(store, to_cfg(tw, cfg)), exp)


def test_c1_walks_all_biases(tw, co, graphs):
    """C1: 100K sampled walks, L=80, every bias, byte-identical."""
    g = graphs["c1"]
    store = tw.EdgeStore.build(g)
    for bias in range(4):
        cfg = Cfg(walk_length=80, start_mode=1, total_walks=100000, bias=bias, seed=7)
        exp, es = co.generate(g, 0, cfg, variant=2)
        st = tw.WalkStats()
        ws = tw.generate_walks(store, to_cfg(tw, cfg), variant=tw.Variant.FullWalk, stats=st)
        assert_walks(ws, exp)
        assert st.hops == es["hops"] and st.ambiguous_draws == 0


def test_walk_sharding_union(tw, graphs):
    """Walk-id shards (multi-GPU partition) concatenate to the full WalkSet."""
    store = tw.EdgeStore.build(graphs["hub"])
    base = tw.WalkConfig(walk_length=20, start_mode=tw.StartMode.Sampled, total_walks=10000, seed=3)
    full = tw.generate_walks(store, base)
    parts = []
    for r in range(4):
        c = tw.WalkConfig(**{**base.__dict__, "walk_begin": r * 2500, "walk_end": (r + 1) * 2500})
        parts.append(tw.generate_walks(store, c))
    assert np.array_equal(np.concatenate([p.nodes for p in parts]), full.nodes)
    assert np.array_equal(np.concatenate([p.times for p in parts]), full.times)


def test_walk_contract_errors(tw):
    s = tw.EdgeStore.build([(1, 2, 1), (2, 3, 2)])
    with pytest.raises(ValueError):
        tw.generate_walks(s, tw.WalkConfig(direction=tw.WalkDirection.Backward))
    with pytest.raises(ValueError):
        tw.generate_walks(s, tw.WalkConfig(start_mode=tw.StartMode.Sampled, total_walks=1 << 40))
    with pytest.raises(ValueError):
        tw.generate_walks(tw.EdgeStore.build([]), tw.WalkConfig(start_mode=tw.StartMode.Sampled, total_walks=3))
    with pytest.raises(ValueError):
        tw.generate_walks(s, tw.WalkConfig(walk_length=0))
    ws = tw.generate_walks(s, tw.WalkConfig(walks_per_node=1, walk_length=3, bias=tw.BiasKind.UniformIndex))
    assert ws.walk_count == 2 and list(ws.lengths) == [3, 2]
    assert [ws.node_at(0, j) for j in range(3)] == [1, 2, 3]
    assert [ws.time_at(0, j) for j in range(3)] == [tw.kTimeUnset, 1, 2]


def test_schedule_step_known_answers(tw):
    """test_walk_engine.cpp:104-136."""
    s = tw.EdgeStore.build([(10, 1, 1), (11, 1, 1), (12, 1, 1)])
    x, y, z = s.find_node(10), s.find_node(11), s.find_node(12)
    cur = [x] * 3 + [y] * 100 + [z] * 20000
    plan = tw.schedule_step(s, cur, [1] * len(cur))
    assert len(plan.solo) == 1 and plan.solo[0].end - plan.solo[0].begin == 3
    assert len(plan.warp_cached) == 1 and plan.warp_cached[0].end - plan.warp_cached[0].begin == 100
    assert [t.end - t.begin for t in plan.block_cached] == [8192, 8192, 3616]
    assert all(t.sub_task_count == 3 for t in plan.block_cached)
    assert not plan.warp_direct and not plan.block_direct


# ------------------------------------------------------------------ samplers

def test_pickers_vs_oracle(tw, co):
    """acceptance.cpp:95-150 style: 10^5 (u, n) pairs, 0 mismatches."""
    rs = np.random.default_rng(31)
    u = rs.random(100000)
    n = rs.integers(1, 10001, 100000).astype(np.uint64)
    ne = rs.integers(1, 701, 100000).astype(np.uint64)
    big = rs.integers(701, 100701, 100000).astype(np.uint64)
    gu = tw.pick_index_uniform(u, n)
    gl = tw.pick_index_linear(u, n)
    ge = tw.pick_index_exponential(u, ne)
    gb = tw.pick_index_exponential(u, big)
    for i in range(100000):
        assert gu[i] == co.pick(0, u[i], int(n[i]))
        assert gl[i] == co.pick(1, u[i], int(n[i]))
        assert ge[i] == co.pick(2, u[i], int(ne[i]))
        assert gb[i] == co.pick(2, u[i], int(big[i]))
    assert tw.pick_index_exponential(1e-300, 100000) == 100000 - 691
    assert tw.pick_index_exponential(0.5, 2) == 1
    assert tw.pick_index_exponential(0.1, 3) == 1
    assert tw.pick_index_linear(0.3, 3) == 1 and tw.pick_index_linear(0.95, 3) == 2
    with pytest.raises(ValueError):
        tw.pick_index_uniform(0.5, 0)


def test_pickers_million_vs_reference(tw, ref):
    """acceptance.cpp:95-150 at its own size: 10^6 random (u, n) per closed
    form against the unmodified reference's pick_index_* (glibc libm on the
    host), 0 mismatches; n spans both exponential regimes (n <= 700 exact
    expm1/log1p form, n > 700 asymptotic form) plus tiny n."""
    rs = np.random.default_rng(1234)
    N = 1_000_000
    u = rs.random(N)
    u[:1000] = np.ldexp(1.0, -rs.integers(1, 1074, 1000).astype(np.int32))  # tiny u (deep tail)
    u[1000:2000] = 1.0 - np.ldexp(1.0, -rs.integers(1, 53, 1000).astype(np.int32))  # u next to 1
    n_all = np.concatenate([rs.integers(1, 16, N // 4), rs.integers(1, 701, N // 4),
                            rs.integers(701, 1 << 20, N // 4), rs.integers(1, 1 << 31, N - 3 * (N // 4))])
    n_all = rs.permutation(n_all).astype(np.uint64)
    got = {0: tw.pick_index_uniform(u, n_all), 1: tw.pick_index_linear(u, n_all),
           2: tw.pick_index_exponential(u, n_all)}
    for kind in (0, 1, 2):
        exp = ref.pick_many(kind, u, n_all)
        bad = np.flatnonzero(np.asarray(got[kind], np.uint64) != exp)
        assert bad.size == 0, (kind, bad[:5], u[bad[:5]], n_all[bad[:5]])


# ------------------------------------------------------------------ replay

def test_replay_parity(tw, co):
    stream = co.gen_uniform(40, 3000, 999, 7)
    stream = stream[np.argsort(stream[:, 2], kind="stable")]
    for bias in (2, 3):
        cfg = Cfg(walk_length=10, start_mode=1, total_walks=500, bias=bias, seed=11)
        exp = co.replay(stream, 100, 333, 0, cfg)
        got = []
        rc = tw.ReplayConfig(batch_duration=100, window_duration=333, walk=to_cfg(tw, cfg))
        n = tw.replay_stream(stream, rc, lambda r, w: got.append((r, w)))
        assert n == len(exp) == 10
        for (r, w), (ei, ew, ex) in zip(got, exp):
            assert (r.ingest.ingested, r.ingest.dropped_late, r.ingest.evicted, r.ingest.retained) == (
                ei["ingested"], ei["dropped_late"], ei["evicted"], ei["retained"])
            assert r.walk.hops == ew["hops"]
            assert_walks(w, ex)


@pytest.mark.parametrize("mode,direction", [(0, 0), (1, 1), (2, 0), (2, 1)])
@pytest.mark.parametrize("t_max", [1000000, 400])
def test_walks_long_runs_bit_exact(tw, co, mode, direction, t_max):
    """Runs of ~200 entries per node (the interpolation search over the
    entries, t_max large: distinct times) and heavily tied runs (the marks,
    t_max small), both walk directions, sampled and per-node starts."""
    g = co.gen_uniform(200, 40000, t_max, 5)
    store = tw.EdgeStore.build(g, tw.DirectionMode(mode))
    for bias in (0, 2):
        for start_mode in (0, 1):
            cfg = Cfg(walk_length=20, start_mode=start_mode, walks_per_node=5, total_walks=4000, bias=bias,
                      seed=13, direction=direction)
            exp, es = co.generate(g, mode, cfg, variant=0)
            st = tw.WalkStats()
            ws = tw.generate_walks(store, to_cfg(tw, cfg), variant=tw.Variant.FullWalk, stats=st)
            assert_walks(ws, exp)
            assert (st.walks, st.hops) == (es["walks"], es["hops"])
