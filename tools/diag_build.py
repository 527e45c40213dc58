import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2605_16182_b200 as tw
from oracle.py import COracle
co = COracle(); ctx = tw.Context(0)
g = co.gen_uniform(100000, 1000000, 1000000, 1)
for w, a in ((True, True), (False, False), (True, True), (False, False), (True, False)):
    for r in range(3):
        ctx.sync(); t0 = time.perf_counter()
        s = tw.EdgeStore.build(g, weights=w, adjacency=a, ctx=ctx)
        ctx.sync(); dt = time.perf_counter() - t0
        print(f"weights={w} adj={a} rep {r}: {dt*1e3:.1f} ms", flush=True)
        del s
