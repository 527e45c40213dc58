"""The GPU causality auditor (csrc/audit.cu, twg_walkset_audit) against the
reference's own EdgeOracle / check_walkset (validity.cpp:14-30, :108-120,
compiled in oracle/_ref): identical (valid walks, walks, valid hops, hops) on
valid walk sets and on walk sets audited against the wrong (later, evicted)
snapshot, for directed / undirected stores and both walk directions."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _walk_dict(ws):
    return dict(stride=ws.stride, walk_count=ws.walk_count, nodes=ws.nodes, times=ws.times, lengths=ws.lengths)


def _stream(co, nodes, edges, tmax, seed):
    g = co.gen_uniform(nodes, edges, tmax, seed)
    return g[np.argsort(g[:, 2], kind="stable")]


def _check(ws, snap, ref, direction=0, undirected=False):
    rep, first = ws.audit(snap, tw_dir(direction), first_violation=True)
    vw, tot_w, vh, tot_h = ref.check_walkset(snap.export_edges(), undirected, _walk_dict(ws), direction)
    assert (rep["valid_walks"], rep["walks"], rep["valid_hops"], rep["hops"]) == (vw, tot_w, vh, tot_h)
    return rep, first


def tw_dir(d):
    import paper_2605_16182_b200 as tw
    return tw.WalkDirection(d)


def test_audit_valid_walks_all_biases(tw, co, ref):
    stream = _stream(co, 3000, 60000, 60000, 5)
    w = tw.WindowManager(20000)
    for off in range(0, len(stream), 6000):
        w.ingest_batch(stream[off:off + 6000])
    snap = w.snapshot()
    for bias in range(4):
        cfg = tw.WalkConfig(start_mode=tw.StartMode.Sampled, total_walks=20000, walk_length=30,
                            bias=tw.BiasKind(bias), seed=3)
        ws = tw.generate_walks(snap, cfg)
        rep, first = _check(ws, snap, ref)
        assert rep["valid_walks"] == rep["walks"] > 0 and rep["valid_hops"] == rep["hops"]
        assert (first == -1).all()


def test_audit_detects_evicted_edges(tw, co, ref):
    """Walks of snapshot k audited against snapshot k+3: hops on evicted edges
    fail; GPU and reference agree on every count, and the first violations
    match a host recomputation."""
    stream = _stream(co, 2000, 40000, 40000, 9)
    w = tw.WindowManager(12000)
    snaps = []
    for off in range(0, len(stream), 4000):
        w.ingest_batch(stream[off:off + 4000])
        snaps.append(w.snapshot())
    cfg = tw.WalkConfig(start_mode=tw.StartMode.Sampled, total_walks=10000, walk_length=20, seed=11)
    ws = tw.generate_walks(snaps[5], cfg)
    rep, first = _check(ws, snaps[8], ref)
    assert rep["valid_hops"] < rep["hops"] and rep["valid_walks"] < rep["walks"]
    # host recomputation of the first violation per walk
    e = snaps[8].export_edges()
    have = set(map(tuple, e.tolist()))
    nodes, times, lens = ws.nodes.reshape(-1, ws.stride), ws.times.reshape(-1, ws.stride), ws.lengths
    for i in range(0, ws.walk_count, 37):
        exp = -1
        for j in range(int(lens[i]) - 1):
            ok = (int(nodes[i, j]), int(nodes[i, j + 1]), int(times[i, j + 1])) in have
            ok = ok and (j == 0 or times[i, j + 1] > times[i, j])
            if not ok:
                exp = j
                break
        assert first[i] == (exp if lens[i] >= 2 else -1), i


@pytest.mark.parametrize("direction", [0, 1])
def test_audit_undirected(tw, co, ref, direction):
    g = co.gen_uniform(500, 8000, 4000, 21)
    snap = tw.EdgeStore.build(g, tw.DirectionMode.Undirected)
    cfg = tw.WalkConfig(start_mode=tw.StartMode.Sampled, total_walks=5000, walk_length=15, seed=2,
                        direction=tw.WalkDirection(direction))
    ws = tw.generate_walks(snap, cfg)
    rep, _ = _check(ws, snap, ref, direction, undirected=True)
    assert rep["valid_hops"] == rep["hops"] > 0


def test_audit_backward_directed(tw, co, ref):
    g = co.gen_uniform(800, 10000, 5000, 4)
    snap = tw.EdgeStore.build(g, tw.DirectionMode.DirectedBackward)
    cfg = tw.WalkConfig(walks_per_node=3, walk_length=12, seed=8, direction=tw.WalkDirection.Backward)
    ws = tw.generate_walks(snap, cfg)
    rep, _ = _check(ws, snap, ref, 1)
    assert rep["valid_hops"] == rep["hops"] > 0
