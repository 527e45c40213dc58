"""Pin the C restatement (oracle/tw_oracle.c) to the compiled, unmodified
reference (oracle/_ref): generators, every index array, window state,
walks for every bias/mode/start/variant, node2vec, Philox, replay, tiers.
CPU only."""
import numpy as np
import pytest

from oracle.py import Cfg

STORE_KEYS = ["src_ext", "dst_ext", "t", "src", "dst", "ts_off", "ts_time", "ts_w", "n_off", "n_tsidx",
              "mk_time", "mk_start", "ref_edge", "wprefix", "ext", "ref_nbr"]
WALK_KEYS = ["nodes", "times", "lengths"]


def assert_store_equal(a, b):
    for k in STORE_KEYS:
        assert np.array_equal(a[k], b[k]), k


def assert_walks_equal(a, b):
    assert a["stride"] == b["stride"] and a["walk_count"] == b["walk_count"]
    for k in WALK_KEYS:
        assert np.array_equal(a[k], b[k]), k


def strip(s):
    s = dict(s)
    s.pop("wall_seconds", None)
    s.pop("rebuild_duration", None)
    s.pop("peak_bytes", None)
    return s


@pytest.fixture(scope="module")
def graphs(co):
    return {
        "uniform": co.gen_uniform(100, 3000, 50, 17),
        "hub": co.gen_hub_skewed(2000, 20000, 0),
        "mega": co.gen_mega_hub(1700, 23),
        "ladder": co.gen_time_ladder(20000, 256, 17),
        "ties": co.gen_uniform(20, 500, 5, 77),
    }


def test_generators_match(co, ref):
    assert np.array_equal(co.gen_uniform(1000, 5000, 999, 3), ref.gen_uniform(1000, 5000, 999, 3))
    assert np.array_equal(co.gen_hub_skewed(300, 3000, 71), ref.gen_hub_skewed(300, 3000, 71))
    assert np.array_equal(co.gen_mega_hub(2500, 55), ref.gen_mega_hub(2500, 55))
    assert np.array_equal(co.gen_time_ladder(1000, 256, 17), ref.gen_time_ladder(1000, 256, 17))


def test_rng_matches(co, ref, ref_philox):
    rs = np.random.default_rng(0)
    for _ in range(200):
        seed, w, h, o = (int(x) for x in rs.integers(0, 2**63, 4))
        assert co.rng_bits(0, seed, w, h, o) == ref.rng_bits(0, seed, w, h, o)
        assert co.rng_bits(1, seed, w, h, o) == ref_philox.rng_bits(1, seed, w, h, o)


@pytest.mark.parametrize("mode", [0, 1, 2])
@pytest.mark.parametrize("name", ["uniform", "hub", "ladder", "ties"])
def test_store_arrays(co, ref, graphs, mode, name):
    assert_store_equal(co.build(graphs[name], mode), ref.build(graphs[name], mode))


def test_store_edge_cases(co, ref):
    big = (1 << 62) + 12345
    for edges in ([], [(7, 8, 3)], [(1, 1, 3), (1, 2, 3), (1, 2, 3)], [(big, big - 7, 1), (big - 7, big, 2)]):
        for mode in (0, 1, 2):
            assert_store_equal(co.build(edges, mode), ref.build(edges, mode))


@pytest.mark.parametrize("mode,direction", [(0, 0), (1, 1), (2, 0), (2, 1)])
@pytest.mark.parametrize("bias", [0, 1, 2, 3])
@pytest.mark.parametrize("start_mode", [0, 1])
def test_walks(co, ref, graphs, mode, direction, bias, start_mode):
    cfg = Cfg(walk_length=12, start_mode=start_mode, walks_per_node=3, total_walks=3000, bias=bias,
              start_bias=(bias + 1) % 4, seed=99, direction=direction)
    for variant in (0, 2):
        a, sa = co.generate(graphs["hub"], mode, cfg, variant=variant)
        b, sb = ref.generate(graphs["hub"], mode, cfg, variant=variant)
        assert_walks_equal(a, b)
        assert strip(sa) == strip(sb)


@pytest.mark.parametrize("temporal", [False, True])
@pytest.mark.parametrize("mode", [0, 2])
def test_node2vec(co, ref, graphs, temporal, mode):
    cfg = Cfg(walk_length=10, start_mode=1, total_walks=4000, bias=3, node2vec=True, p=0.5, q=2.0,
              temporal_adjacency=temporal, seed=7)
    a, _ = co.generate(graphs["uniform"], mode, cfg)
    b, _ = ref.generate(graphs["uniform"], mode, cfg)
    assert_walks_equal(a, b)


def test_philox_walks(co, ref_philox, graphs):
    for bias in range(4):
        cfg = Cfg(walk_length=16, start_mode=1, total_walks=3000, bias=bias, seed=5, rng=1)
        a, _ = co.generate(graphs["hub"], 0, cfg)
        b, _ = ref_philox.generate(graphs["hub"], 0, cfg)
        assert_walks_equal(a, b)


def test_tier_counts_c3b(co, ref, graphs):
    """acceptance criterion 6 (acceptance.cpp:276-294; test_output.txt:38)."""
    a, sa = co.generate(graphs["hub"], 0, Cfg())
    b, sb = ref.generate(graphs["hub"], 0, Cfg())
    assert strip(sa) == strip(sb)
    assert (sa["solo"], sa["warp_cached"], sa["warp_direct"], sa["block_cached"], sa["block_direct"],
            sa["multi_block"]) == (19, 6230, 4, 11, 1, 7)


def test_window_sequence(co, ref):
    rs = np.random.default_rng(3)
    batches, base = [], 0
    for b in range(12):
        n = 400
        t = base + rs.integers(0, 40, n)
        batches.append(np.stack([rs.integers(0, 30, n), rs.integers(0, 30, n), t], 1))
        base += 25
    batches.insert(5, np.zeros((0, 3), np.int64))
    for mode in (0, 2):
        sa, da = co.window_run(batches, 50, mode)
        sb, db = ref.window_run(batches, 50, mode)
        assert [(strip(x), y) for x, y in sa] == [(strip(x), y) for x, y in sb]
        assert_store_equal(da, db)


def test_replay(co, ref):
    stream = co.gen_uniform(40, 3000, 999, 7)
    stream = stream[np.argsort(stream[:, 2], kind="stable")]
    for bias in (2, 3):
        cfg = Cfg(walk_length=10, start_mode=1, total_walks=500, bias=bias, seed=11)
        ra = co.replay(stream, 100, 333, 0, cfg)
        rb = ref.replay(stream, 100, 333, 0, cfg)
        assert len(ra) == len(rb) == 10
        for (ia, wa, xa), (ib, wb, xb) in zip(ra, rb):
            assert strip(ia) == strip(ib)
            assert strip(wa) == strip(wb)
            assert_walks_equal(xa, xb)
