"""Diagnostic: GPU causality audit of one C5 walk generation (10M walks) on
the steady-state window (device-timed), and its report."""
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
cfg = tw.WalkConfig(walk_length=80, start_mode=tw.StartMode.Sampled, total_walks=wl.walks,
                    bias=tw.BiasKind.ExponentialIndex, seed=5)
ws = tw.generate_walks(snap, cfg, variant=tw.Variant.FullWalk)
for r in range(2):
    ctx.sync()
    t0 = time.perf_counter()
    rep, _ = ws.audit(snap)
    print(f"audit rep {r}: {(time.perf_counter() - t0) * 1e3:.1f} ms {rep}", flush=True)
