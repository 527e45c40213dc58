"""Diagnostic: walk-phase time on the C5 window by walk length (L=3: the start
edge + one causal search from a uniform time; L=80: the full walk), to split
the first-hop search cost from the later hops'. usage: diag_walk_len.py"""
import sys
import time

sys.path.insert(0, ".")
import torch

import paper_2605_16182_b200 as tw
from bench import Workload

wl = Workload(1.0)
ctx = tw.Context(0)
lib = tw._abi.load()
B = wl.batch_edges
w = tw.WindowManager(wl.window, weights=False, adjacency=False, ctx=ctx)
dev = [torch.empty(B, dtype=torch.int64, device="cuda") for _ in range(3)]
for b in range(wl.prefill + 1):
    lib.twg_synth_stream_device(ctx.handle, wl.nodes, b * B, B, wl.seed, dev[0].data_ptr(), dev[1].data_ptr(),
                                dev[2].data_ptr())
    w.ingest_batch_device(dev[0].data_ptr(), dev[1].data_ptr(), dev[2].data_ptr(), B, stats=False)
snap = w.snapshot()
for L in (2, 3, 4, 80):
    cfg = tw.WalkConfig(walk_length=L, start_mode=tw.StartMode.Sampled, total_walks=wl.walks,
                        bias=tw.BiasKind.ExponentialIndex, seed=5)
    best = None
    for r in range(3):
        ctx.sync()
        t0 = time.perf_counter()
        st = tw.WalkStats()
        ws = tw.generate_walks(snap, cfg, variant=tw.Variant.FullWalk, stats=st)
        ctx.sync()
        dt = (time.perf_counter() - t0) * 1e3
        best = dt if best is None else min(best, dt)
        del ws
    print(f"L={L:3d}: {best:7.3f} ms hops {st.hops}", flush=True)
