"""Generate the golden fixtures from the UNMODIFIED reference (oracle/_ref).

Run in the dev container (needs oracle/_ref built from /root/reference):
    python tests/golden/make_golden.py
Writes tests/golden/golden.npz (committed). The fixtures pin the CPU
restatement and the GPU path even where oracle/_ref is absent.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.py import Cfg, RefOracle  # noqa: E402

KEYS = ["src_ext", "dst_ext", "t", "src", "dst", "ts_off", "ts_time", "ts_w", "n_off", "n_tsidx", "mk_time",
        "mk_start", "ref_edge", "wprefix", "ext", "ref_nbr"]


def graphs(ref):
    return {
        "uniform": ref.gen_uniform(100, 3000, 50, 17),
        "hub": ref.gen_hub_skewed(2000, 20000, 0),
        "ties": ref.gen_uniform(20, 500, 5, 77),
    }


WALK_CASES = [  # (graph, mode, cfg kwargs, variant)
    ("hub", 0, dict(walk_length=12, start_mode=0, walks_per_node=2, bias=3, seed=99), 0),
    ("hub", 0, dict(walk_length=20, start_mode=1, total_walks=2000, bias=0, seed=7), 2),
    ("hub", 0, dict(walk_length=20, start_mode=1, total_walks=2000, bias=1, start_bias=2, seed=7), 2),
    ("hub", 0, dict(walk_length=20, start_mode=1, total_walks=2000, bias=2, start_bias=3, seed=7), 2),
    ("uniform", 1, dict(walk_length=10, start_mode=0, walks_per_node=3, bias=3, direction=1, seed=5), 0),
    ("uniform", 2, dict(walk_length=10, start_mode=1, total_walks=2000, bias=3, node2vec=True, p=0.5, q=2.0,
                        seed=7), 0),
    ("uniform", 2, dict(walk_length=10, start_mode=1, total_walks=2000, bias=3, node2vec=True, p=0.25, q=4.0,
                        temporal_adjacency=True, seed=3), 0),
]
PHILOX_CASES = [("hub", 0, dict(walk_length=16, start_mode=1, total_walks=2000, bias=b, seed=5, rng=1), 0)
                for b in range(4)]


def main():
    ref = RefOracle()
    refp = RefOracle(philox=True)
    g = graphs(ref)
    out = {}
    for name, e in g.items():
        out[f"graph/{name}"] = e
        for mode in (0, 1, 2):
            d = ref.build(e, mode)
            for k in KEYS:
                out[f"store/{name}/{mode}/{k}"] = d[k]
    for i, (gname, mode, kw, var) in enumerate(WALK_CASES + PHILOX_CASES):
        r = refp if kw.get("rng") == 1 else ref
        w, st = r.generate(g[gname], mode, Cfg(**kw), variant=var)
        for k in ("nodes", "times", "lengths"):
            out[f"walk/{i}/{k}"] = w[k]
        out[f"walk/{i}/stride"] = np.array([w["stride"]])
        out[f"walk/{i}/stats"] = np.array([st["walks"], st["hops"], st["steps"], st["solo"], st["warp_cached"],
                                           st["warp_direct"], st["block_cached"], st["block_direct"],
                                           st["multi_block"]], np.uint64)
    # window sequence (stats after every batch + final state)
    rs = np.random.default_rng(3)
    batches, base = [], 0
    for b in range(10):
        n = 300
        batches.append(np.stack([rs.integers(0, 30, n), rs.integers(0, 30, n), base + rs.integers(0, 40, n)], 1))
        base += 25
    stats, d = ref.window_run(batches, 50, 0)
    for i, b in enumerate(batches):
        out[f"window/batch/{i}"] = b
    out["window/stats"] = np.array([[s["ingested"], s["dropped_late"], s["evicted"], s["retained"],
                                     bnd[0], bnd[1]] for s, bnd in stats], np.int64)
    for k in KEYS:
        out[f"window/final/{k}"] = d[k]
    # pickers on a sweep (samplers.cpp:17-55)
    rs = np.random.default_rng(31)
    u = rs.random(20000)
    n = rs.integers(1, 5001, 20000).astype(np.uint64)
    ne = rs.integers(1, 1501, 20000).astype(np.uint64)
    out["pick/u"] = u
    out["pick/n"] = n
    out["pick/ne"] = ne
    out["pick/uniform"] = ref.pick_many(0, u, n)
    out["pick/linear"] = ref.pick_many(1, u, n)
    out["pick/exponential"] = ref.pick_many(2, u, ne)
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
