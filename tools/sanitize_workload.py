"""A small end-to-end workload for compute-sanitizer (tests/test_gpu_sanitizer.py):
the streaming append route (ring relocations, arena repacks, the onesweep
look-back, tie merges) in all three direction modes, the general rebuild
route, and every walk variant (Coop / CoopDirect / FullWalk, all biases,
node2vec) plus the auditor and the walk writers. No torch: only the C ABI
through the package's ctypes mirror, so the sanitizer sees our kernels alone.

usage: compute-sanitizer --tool memcheck python tools/sanitize_workload.py
       TWG_GUARD=1 python tools/sanitize_workload.py   (poisoned blocks + tail guards)

Prints a digest of every walk set it downloads, so a poisoned run (TWG_GUARD=1:
fresh device blocks filled with 0xA5) can be compared with a plain one.
"""
import gc
import hashlib
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_16182_b200 as tw  # noqa: E402


def stream(seed, nb, n, nodes, step, tie_boundary=False):
    rs = np.random.default_rng(seed)
    out, last_t = [], None
    for b in range(nb):
        t = np.sort(b * step + rs.integers(0, step, n))
        s = rs.integers(0, nodes, n)
        d = np.minimum((nodes * rs.random(n) ** 3).astype(np.int64), nodes - 1)
        e = np.stack([s, d, t], 1)
        e = e[np.lexsort((e[:, 1], e[:, 0], e[:, 2]))]
        if tie_boundary and last_t is not None:
            e[0] = (nodes - 1, nodes - 1, last_t)
        last_t = int(e[-1, 2])
        out.append(e)
    return out


def main():
    h = hashlib.sha256()

    def take(ws):
        for a in (ws.nodes, ws.times, ws.lengths):
            h.update(memoryview(a).cast("B"))

    for mode in (0, 1, 2):
        w = tw.WindowManager(250, tw.DirectionMode(mode))
        for b in stream(40 + mode, 10, 1500, 120, 100, tie_boundary=mode == 2):
            w.ingest_batch(b)
        snap = w.snapshot()
        assert snap.is_streaming()
        dirs = [0, 1] if mode == 2 else [0 if mode == 0 else 1]
        for d in dirs:
            for variant in (tw.Variant.Coop, tw.Variant.CoopDirect, tw.Variant.FullWalk):
                for bias in (tw.BiasKind.UniformIndex, tw.BiasKind.ExponentialIndex, tw.BiasKind.ExponentialWeight):
                    cfg = tw.WalkConfig(walk_length=12, start_mode=tw.StartMode.Sampled, total_walks=600, bias=bias,
                                        start_bias=bias, direction=tw.WalkDirection(d), seed=3)
                    ws = tw.generate_walks(snap, cfg, variant=variant)
                    take(ws)
            cfg = tw.WalkConfig(walk_length=10, start_mode=tw.StartMode.PerNode, walks_per_node=2,
                                bias=tw.BiasKind.ExponentialWeight, direction=tw.WalkDirection(d), seed=5,
                                node2vec=tw.Node2VecParams(0.5, 2.0))
            ws = tw.generate_walks(snap, cfg)
            take(ws)
            h.update(repr(ws.audit(snap, direction=tw.WalkDirection(d))).encode())
    # general route (unordered batch) + EdgeStore::build + hub tiers
    g = tw.synth_graph("hub_skewed", 2000, 20000, seed=0)
    st = tw.EdgeStore.build(g)
    ws = tw.generate_walks(st, tw.WalkConfig())
    take(ws)
    w = tw.WindowManager(10 ** 9)
    w.ingest_batch(g[::-1].copy())
    take(tw.generate_walks(w.snapshot(), tw.WalkConfig(seed=9)))
    del w, ws, st, snap
    gc.collect()  # device blocks freed (and, under TWG_GUARD, their guards checked) before the digest
    print("digest", h.hexdigest())
    print("sanitize workload ok")


if __name__ == "__main__":
    main()
