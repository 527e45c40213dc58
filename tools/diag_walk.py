"""Diagnostic: C5-shaped window at a given scale, then timed walk generation
(CUDA events on the library stream), per variant."""
import sys
import time

sys.path.insert(0, ".")
import torch

import paper_2605_16182_b200 as tw
from bench import Workload

scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
variants = sys.argv[3].split(",") if len(sys.argv) > 3 else ["fullwalk"]
walk_length = int(sys.argv[4]) if len(sys.argv) > 4 else 80
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
print("window edges", snap.edge_count(), "nodes", snap.node_count(), flush=True)
stream = torch.cuda.ExternalStream(ctx.stream)
cfg = tw.WalkConfig(walk_length=walk_length, start_mode=tw.StartMode.Sampled, total_walks=wl.walks,
                    bias=tw.BiasKind.ExponentialIndex, seed=5)
for v in variants:
    var = {"fullwalk": tw.Variant.FullWalk, "coop": tw.Variant.Coop, "coopdirect": tw.Variant.CoopDirect}[v]
    for r in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ctx.sync()
        t0 = time.perf_counter()
        e0.record(stream)
        st = tw.WalkStats()
        ws = tw.generate_walks(snap, cfg, variant=var, stats=st)
        e1.record(stream)
        ctx.sync()
        dt = time.perf_counter() - t0
        print(f"{v:10s} rep {r}: events {e0.elapsed_time(e1):8.2f} ms wall {dt*1e3:8.2f} ms hops {st.hops} "
              f"steps {st.steps} alg {st.alg_bytes/1e9:.2f} GB amb {st.ambiguous_draws}", flush=True)
        del ws
