"""The reference's acceptance criteria (proj/tests/acceptance.cpp) restated
against the GPU path, for BOTH RNG streams: with SplitMix the walks are the
reference's byte for byte; with Philox they are a different but equally
valid random stream, checked distributionally at stated significance
(north_star: chi-square / total-variation tests) and for causality."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

RNGS = ["SplitMix", "Philox"]


def chi2_sf(x, dof):
    """Chi-square survival function (regularised upper incomplete gamma)."""
    from scipy.special import gammaincc
    return float(gammaincc(dof / 2.0, x / 2.0))


def tv(counts, probs):
    counts = np.asarray(counts, dtype=np.float64)
    return 0.5 * float(np.abs(counts / counts.sum() - np.asarray(probs)).sum())


@pytest.mark.parametrize("rng", RNGS)
def test_causality_soundness(tw, co, ref, rng):
    """acceptance.cpp:52-91: 100% of hops/walks causality-valid, 4 biases,
    100K walks each, window over a 10-batch 1M-edge stream (audited by the
    reference's own EdgeOracle/check_walkset)."""
    stream = co.gen_uniform(50000, 1000000, 1000000, 2024)
    stream = stream[np.argsort(stream[:, 2], kind="stable")]
    w = tw.WindowManager(300000)
    for off in range(0, len(stream), 100000):
        w.ingest_batch(stream[off:off + 100000])
    snap = w.snapshot()
    edges = snap.export_edges()
    for bias in range(4):
        cfg = tw.WalkConfig(start_mode=tw.StartMode.Sampled, total_walks=100000, walk_length=80,
                            bias=tw.BiasKind(bias), seed=7, rng=tw.RngKind[rng])
        ws = tw.generate_walks(snap, cfg)
        walks = dict(stride=ws.stride, walk_count=ws.walk_count, nodes=ws.nodes, times=ws.times,
                     lengths=ws.lengths)
        vw, tw_, vh, th = ref.check_walkset(edges, False, walks)
        assert vw == tw_ and vh == th and tw_ > 0


@pytest.mark.parametrize("rng", RNGS)
def test_weighted_sampler_tv(tw, rng):
    """acceptance.cpp:154-186: exp-weight picks over a 16-edge neighbourhood
    with irregular gaps, 10^6 draws, TV < 0.01."""
    times = [0, 1, 3, 4, 7, 11, 12, 13, 20, 22, 23, 25, 26, 30, 33, 37]
    edges = [(0, 100 + i, t) for i, t in enumerate(times)]
    store = tw.EdgeStore.build(edges)
    cfg = tw.WalkConfig(walks_per_node=1000000, walk_length=2, bias=tw.BiasKind.ExponentialWeight, seed=12,
                        rng=tw.RngKind[rng])
    ws = tw.generate_walks(store, cfg, variant=tw.Variant.FullWalk)
    ln = ws.lengths
    picked = ws.nodes.reshape(-1, ws.stride)[ln >= 2, 1] - 100
    counts = np.bincount(picked, minlength=len(times))
    w = np.exp(np.array(times, dtype=np.float64) - times[0])
    p = w / w.sum()
    assert tv(counts, p) < 0.01
    # chi-square on cells with expected count >= 5
    exp = p * counts.sum()
    keep = exp >= 5
    stat = float(((counts[keep] - exp[keep]) ** 2 / exp[keep]).sum())
    assert chi2_sf(stat, keep.sum() - 1) > 1e-3


@pytest.mark.parametrize("rng", RNGS)
def test_node2vec_rejection_tv(tw, rng):
    """acceptance.cpp:190-231: node2vec second-order transitions out of C
    after S->C@1 for (p,q) in {(0.5,2), (2,0.5), (1,1)}: TV < 0.02."""
    S, C_, A, B = 1, 2, 3, 4
    edges = [(S, C_, 1), (C_, S, 2), (S, A, 2), (C_, A, 3), (C_, B, 5)]
    store = tw.EdgeStore.build(edges)
    for p, q in [(0.5, 2.0), (2.0, 0.5), (1.0, 1.0)]:
        n_s = n_a = n_b = kept = 0
        for rnd in range(5):
            cfg = tw.WalkConfig(start_mode=tw.StartMode.Sampled, total_walks=1200000, walk_length=3,
                                bias=tw.BiasKind.ExponentialWeight, node2vec=tw.Node2VecParams(p, q),
                                seed=1000 + rnd, rng=tw.RngKind[rng])
            ws = tw.generate_walks(store, cfg, variant=tw.Variant.FullWalk)
            nodes = ws.nodes.reshape(-1, ws.stride)
            sel = (ws.lengths >= 3) & (nodes[:, 1] == C_)
            hop = nodes[sel, 2][: 1000000 - kept]
            kept += len(hop)
            n_s += int((hop == S).sum())
            n_a += int((hop == A).sum())
            n_b += int((hop == B).sum())
            if kept >= 1000000:
                break
        expected = np.array([1.0 / p, math.e, math.exp(3.0) / q])
        expected /= expected.sum()
        assert tv([n_s, n_a, n_b], expected) < 0.02, (p, q, n_s, n_a, n_b)


@pytest.mark.parametrize("rng", RNGS)
def test_exponential_index_chi_square(tw, rng):
    """acceptance.cpp:124-148: the asymptotic exponential picker (n = 1000,
    10000) against its analytic e^i mass, top-12 indices + tail, p > 1e-3."""
    bits = tw.rng_bits(tw.RngKind[rng], 31, np.arange(1000000, dtype=np.uint64), 3, 0)
    u = (bits >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    for n in (1000, 10000):
        idx = tw.pick_index_exponential(u, n).astype(np.int64)
        j = n - 1 - idx
        obs = np.bincount(np.minimum(j, 12), minlength=13)
        norm = (1 - math.exp(-1)) / (1 - math.exp(-n))
        exp = np.array([1e6 * math.exp(-k) * norm for k in range(12)])
        exp = np.append(exp, 1e6 - exp.sum())
        stat = float(((obs - exp) ** 2 / exp).sum())
        assert chi2_sf(stat, 12) > 1e-3


@pytest.mark.parametrize("bias", [0, 1, 2])
def test_index_bias_per_hop_distribution_philox(tw, bias):
    """Per-hop transition distribution of Philox walks against the analytic
    index-bias law (uniform / linear / exponential over a node's n = 8
    candidates), chi-square p > 1e-3 at 2*10^5 draws."""
    n = 8
    edges = [(0, 100 + i, i + 1) for i in range(n)]  # node 0: 8 candidates at distinct times
    store = tw.EdgeStore.build(edges)
    cfg = tw.WalkConfig(walks_per_node=200000, walk_length=2, bias=tw.BiasKind(bias), seed=3,
                        rng=tw.RngKind.Philox)
    ws = tw.generate_walks(store, cfg, variant=tw.Variant.FullWalk)
    nodes = ws.nodes.reshape(-1, ws.stride)
    picked = nodes[ws.lengths >= 2, 1] - 100
    obs = np.bincount(picked, minlength=n).astype(np.float64)
    k = np.arange(n, dtype=np.float64)
    w = {0: np.ones(n), 1: k + 1, 2: np.exp(k)}[bias]
    exp = w / w.sum() * obs.sum()
    keep = exp >= 5
    stat = float(((obs[keep] - exp[keep]) ** 2 / exp[keep]).sum())
    assert chi2_sf(stat, keep.sum() - 1) > 1e-3
