"""Golden fixtures made by the unmodified reference (tests/golden/make_golden.py
over oracle/_ref): pin the CPU restatement (CPU test) and the GPU path
(gpu test) even where oracle/_ref is not present."""
import os

import numpy as np
import pytest

from oracle.py import Cfg

HERE = os.path.dirname(os.path.abspath(__file__))
G = np.load(os.path.join(HERE, "golden", "golden.npz"))
KEYS = ["src_ext", "dst_ext", "t", "src", "dst", "ts_off", "ts_time", "ts_w", "n_off", "n_tsidx", "mk_time",
        "mk_start", "ref_edge", "wprefix", "ext", "ref_nbr"]

from tests.golden.make_golden import PHILOX_CASES, WALK_CASES  # noqa: E402

CASES = WALK_CASES + PHILOX_CASES


def _eq(a, b):
    a, b = np.asarray(a), np.asarray(b)
    if a.dtype.kind == "f":
        return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.astype(np.float64).view(np.uint64))
    return a.shape == b.shape and np.array_equal(a.astype(np.int64), b.astype(np.int64))


@pytest.mark.parametrize("name", ["uniform", "hub", "ties"])
@pytest.mark.parametrize("mode", [0, 1, 2])
def test_oracle_store_golden(co, name, mode):
    d = co.build(G[f"graph/{name}"], mode)
    for k in KEYS:
        assert _eq(d[k], G[f"store/{name}/{mode}/{k}"]), k


@pytest.mark.parametrize("i", range(len(CASES)))
def test_oracle_walks_golden(co, i):
    gname, mode, kw, var = CASES[i]
    w, st = co.generate(G[f"graph/{gname}"], mode, Cfg(**kw), variant=var)
    for k in ("nodes", "times", "lengths"):
        assert _eq(w[k], G[f"walk/{i}/{k}"]), k
    s = G[f"walk/{i}/stats"]
    assert [st["walks"], st["hops"], st["steps"], st["solo"], st["warp_cached"], st["warp_direct"],
            st["block_cached"], st["block_direct"], st["multi_block"]] == [int(x) for x in s]


def test_oracle_window_golden(co):
    batches = [G[f"window/batch/{i}"] for i in range(10)]
    stats, d = co.window_run(batches, 50, 0)
    got = np.array([[s["ingested"], s["dropped_late"], s["evicted"], s["retained"], b[0], b[1]]
                    for s, b in stats], np.int64)
    assert np.array_equal(got, G["window/stats"])
    for k in KEYS:
        assert _eq(d[k], G[f"window/final/{k}"]), k


def test_oracle_pickers_golden(co):
    u, n, ne = G["pick/u"], G["pick/n"], G["pick/ne"]
    for i in range(0, len(u), 7):
        assert co.pick(0, u[i], int(n[i])) == G["pick/uniform"][i]
        assert co.pick(1, u[i], int(n[i])) == G["pick/linear"][i]
        assert co.pick(2, u[i], int(ne[i])) == G["pick/exponential"][i]


# ---------------------------------------------------------------- GPU vs golden

@pytest.mark.gpu
@pytest.mark.parametrize("name", ["uniform", "hub", "ties"])
@pytest.mark.parametrize("mode", [0, 1, 2])
def test_gpu_store_golden(tw, name, mode):
    d = tw.EdgeStore.build(G[f"graph/{name}"], tw.DirectionMode(mode)).dump(KEYS)
    for k in KEYS:
        assert _eq(d[k], G[f"store/{name}/{mode}/{k}"]), k


@pytest.mark.gpu
@pytest.mark.parametrize("i", range(len(CASES)))
def test_gpu_walks_golden(tw, i):
    gname, mode, kw, var = CASES[i]
    c = Cfg(**kw)
    cfg = tw.WalkConfig(walk_length=c.walk_length, start_mode=tw.StartMode(c.start_mode),
                        walks_per_node=c.walks_per_node, total_walks=c.total_walks, bias=tw.BiasKind(c.bias),
                        start_bias=tw.BiasKind(c.start_bias), node2vec=tw.Node2VecParams(c.p, c.q) if c.node2vec else None,
                        node2vec_temporal_adjacency=c.temporal_adjacency, direction=tw.WalkDirection(c.direction),
                        seed=c.seed, rng=tw.RngKind(c.rng))
    store = tw.EdgeStore.build(G[f"graph/{gname}"], tw.DirectionMode(mode))
    ws = tw.generate_walks(store, cfg, variant=tw.Variant(var))
    assert _eq(ws.nodes, G[f"walk/{i}/nodes"]) and _eq(ws.times, G[f"walk/{i}/times"])
    assert _eq(ws.lengths, G[f"walk/{i}/lengths"])


@pytest.mark.gpu
def test_gpu_window_golden(tw):
    w = tw.WindowManager(50)
    for i in range(10):
        st = w.ingest_batch(G[f"window/batch/{i}"])
        row = G["window/stats"][i]
        assert [st.ingested, st.dropped_late, st.evicted, st.retained, *w.window_bounds()] == [int(x) for x in row]
    d = w.snapshot().dump(KEYS)
    for k in KEYS:
        assert _eq(d[k], G[f"window/final/{k}"]), k


@pytest.mark.gpu
def test_gpu_pickers_golden(tw):
    u, n, ne = G["pick/u"], G["pick/n"], G["pick/ne"]
    assert np.array_equal(tw.pick_index_uniform(u, n), G["pick/uniform"])
    assert np.array_equal(tw.pick_index_linear(u, n), G["pick/linear"])
    assert np.array_equal(tw.pick_index_exponential(u, ne), G["pick/exponential"])
