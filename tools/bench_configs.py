"""BASELINE.json configs C1-C4 on one B200 (C5 is bench.py): build / ingest
time and walk steps/s per config, device-timed (wall clock with a device sync on both
sides). Inputs come from the reference's own counter-based generators
(oracle C restatement, bit-identical to synthetic.cpp). Prints one JSON line
per measurement; tools/bench_configs.py > gpurun_out/configs.jsonl"""
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2605_16182_b200 as tw
from oracle.py import COracle

co = COracle()
ctx = tw.Context(0)
stream = torch.cuda.ExternalStream(ctx.stream)
only = sys.argv[1].split(",") if len(sys.argv) > 1 else ["C1", "C2", "C3", "C4"]


def timed(fn, reps=1):
    """wall time with a device sync on both sides (min over reps; the result of the last rep)"""
    best = None
    for _ in range(reps):
        ctx.sync()
        t0 = time.perf_counter()
        r = fn()
        ctx.sync()
        ms = (time.perf_counter() - t0) * 1e3
        best = ms if best is None else min(best, ms)
    return r, best


def walks(store, cfg, variant=tw.Variant.FullWalk, reps=2):
    best = None
    for _ in range(reps):
        st = tw.WalkStats()
        ws, ms = timed(lambda: tw.generate_walks(store, cfg, variant=variant, stats=st))
        del ws
        best = ms if best is None else min(best, ms)
    return st, best


def emit(**kw):
    print(json.dumps(kw), flush=True)


# warm-up: module load, pools, first-launch costs stay out of the numbers
_w = tw.EdgeStore.build(co.gen_uniform(1000, 10000, 10000, 3), ctx=ctx)
tw.generate_walks(_w, tw.WalkConfig(start_mode=tw.StartMode.Sampled, total_walks=1000, walk_length=8))
_ww = tw.WindowManager(5000, ctx=ctx)
_ww.ingest_batch(co.gen_uniform(1000, 10000, 10000, 3))
del _w, _ww

BIAS = {"uniform": tw.BiasKind.UniformIndex, "linear": tw.BiasKind.LinearIndex,
        "exp_index": tw.BiasKind.ExponentialIndex, "exp_weight": tw.BiasKind.ExponentialWeight}

if "C1" in only:
    g = co.gen_uniform(100000, 1000000, 1000000, 1)
    store, ms = timed(lambda: tw.EdgeStore.build(g, ctx=ctx), reps=3)
    emit(config="C1", what="build 1M edges from host (H2D + weights + adjacency)", ms=ms,
         edges_per_s=len(g) / ms * 1e3)
    for name, b in BIAS.items():
        cfg = tw.WalkConfig(start_mode=tw.StartMode.Sampled, total_walks=100000, walk_length=80, bias=b,
                            start_bias=tw.BiasKind.UniformIndex, seed=7)
        st, ms = walks(store, cfg)
        emit(config="C1", what=f"100K sampled walks L=80 {name}", ms=ms, hops=st.hops, steps_per_s=st.hops / ms * 1e3)

if "C2" in only:
    g = co.gen_uniform(100000, 1000000, 1000000, 1)
    g = g[np.argsort(g[:, 2], kind="stable")]
    bounds = tw.split_batches(g[:, 2], 100000)
    for name in ("exp_weight", "exp_index", "exp_weight"):  # the first pass also warms the pools
        w = tw.WindowManager(333333, ctx=ctx)
        ing = wk = hops = 0.0
        for k, (a, b) in enumerate(bounds):
            _, ms = timed(lambda: w.ingest_batch(g[a:b]))
            ing += ms
            cfg = tw.WalkConfig(start_mode=tw.StartMode.Sampled, total_walks=100000, walk_length=80, bias=BIAS[name],
                                seed=7 + k)
            st, ms = walks(w.snapshot(), cfg, reps=1)
            wk += ms
            hops += st.hops
        emit(config="C2", what=f"10-batch replay, window 333333, 100K walks/batch {name} (host batches)",
             ingest_ms=ing, walk_ms=wk, steps_per_s=hops / (ing + wk) * 1e3, walk_steps_per_s=hops / wk * 1e3)

if "C3" in only:
    t0 = time.perf_counter()
    g = co.gen_hub_skewed(10000000, 100000000, 1)
    gen_s = time.perf_counter() - t0
    store, ms = timed(lambda: tw.EdgeStore.build(g, weights=False, adjacency=False, ctx=ctx))
    emit(config="C3", what=f"build {len(g)} hub-skewed edges (host generation {gen_s:.1f} s)", ms=ms,
         edges_per_s=len(g) / ms * 1e3)
    cfg = tw.WalkConfig(start_mode=tw.StartMode.Sampled, total_walks=10000000, walk_length=80,
                        bias=tw.BiasKind.LinearIndex, seed=7)
    for vname, v in (("fullwalk", tw.Variant.FullWalk), ("coop", tw.Variant.Coop)):
        st, ms = walks(store, cfg, v)
        emit(config="C3", what=f"10M sampled walks L=80 linear {vname}", ms=ms, hops=st.hops,
             steps_per_s=st.hops / ms * 1e3,
             tiers=[st.tiers.solo, st.tiers.warp_cached, st.tiers.warp_direct, st.tiers.block_cached,
                    st.tiers.block_direct, st.tiers.multi_block] if vname == "coop" else None)
    del store, g

if "C4" in only:
    t0 = time.perf_counter()
    g = co.gen_uniform(10000000, 100000000, 99999999, 4)
    gen_s = time.perf_counter() - t0
    store, ms = timed(lambda: tw.EdgeStore.build(g, tw.DirectionMode.Undirected, ctx=ctx))
    emit(config="C4", what=f"build 100M undirected edges + weights + adjacency (host generation {gen_s:.1f} s)",
         ms=ms, edges_per_s=len(g) / ms * 1e3)
    cfg = tw.WalkConfig(start_mode=tw.StartMode.Sampled, total_walks=10000000, walk_length=80,
                        bias=tw.BiasKind.ExponentialWeight, node2vec=tw.Node2VecParams(0.5, 2.0), seed=7)
    st, ms = walks(store, cfg)
    emit(config="C4", what="10M start-edge walks L=80 temporal node2vec (p=0.5, q=2) exp-weight", ms=ms,
         hops=st.hops, steps_per_s=st.hops / ms * 1e3)
