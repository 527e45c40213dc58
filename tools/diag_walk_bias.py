"""Diagnostic: walk generation time per bias on the C5 steady-state window
(streaming snapshot; exp-weight evaluated without materialised prefixes)."""
import sys
import time

sys.path.insert(0, ".")
import torch

import paper_2605_16182_b200 as tw
from bench import Workload

scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
wl = Workload(scale)
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
print("streaming snapshot:", snap.is_streaming(), flush=True)
for name, bias, sb in (("exp_index", 2, 0), ("exp_weight", 3, 0), ("exp_weight+start", 3, 3), ("uniform", 0, 0),
                       ("linear", 1, 0)):
    cfg = tw.WalkConfig(walk_length=80, start_mode=tw.StartMode.Sampled, total_walks=wl.walks,
                        bias=tw.BiasKind(bias), start_bias=tw.BiasKind(sb), seed=5)
    for r in range(2):
        ctx.sync()
        t0 = time.perf_counter()
        st = tw.WalkStats()
        ws = tw.generate_walks(snap, cfg, variant=tw.Variant.FullWalk, stats=st)
        ctx.sync()
        dt = time.perf_counter() - t0
        del ws
    print(f"{name:18s} {dt*1e3:8.2f} ms  hops {st.hops}  {st.hops/dt/1e9:.2f} G steps/s", flush=True)
