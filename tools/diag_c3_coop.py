"""Diagnostic: C3 (hub-skewed 100M edges, linear bias, 10M sampled walks) walk
generation with the cooperative scheduler and with FullWalk (for ncu captures
of the tier kernels)."""
import sys
import time

sys.path.insert(0, ".")
import paper_2605_16182_b200 as tw
from oracle.py import COracle

co = COracle()
ctx = tw.Context(0)
g = co.gen_hub_skewed(10000000, 100000000, 1)
store = tw.EdgeStore.build(g, weights=False, adjacency=False, ctx=ctx)
del g
cfg = tw.WalkConfig(start_mode=tw.StartMode.Sampled, total_walks=10000000, walk_length=80,
                    bias=tw.BiasKind.LinearIndex, seed=7)
variants = [tw.Variant(int(x)) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [tw.Variant.Coop, tw.Variant.CoopDirect, tw.Variant.FullWalk]
for v in variants:
    for r in range(2):
        ctx.sync()
        t0 = time.perf_counter()
        st = tw.WalkStats()
        ws = tw.generate_walks(store, cfg, variant=v, stats=st)
        ctx.sync()
        print(v, f"{(time.perf_counter() - t0) * 1e3:.2f} ms", st.hops, flush=True)
        del ws
