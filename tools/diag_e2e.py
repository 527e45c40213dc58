"""Per-phase wall times of the pipelined e2e loop (bench.run_e2e_pipelined)."""
import ctypes as C
import sys
import time

sys.path.insert(0, ".")
import torch

import paper_2605_16182_b200 as tw
from bench import Workload

wl = Workload(float(sys.argv[1]) if len(sys.argv) > 1 else 1.0)
mode = sys.argv[2] if len(sys.argv) > 2 else "pipe"
ctx = tw.Context(0)
lib = tw._abi.load()
B = wl.batch_edges
w = tw.WindowManager(wl.window, weights=False, adjacency=False, ctx=ctx)
dev = [torch.empty(B, dtype=torch.int64, device="cuda") for _ in range(3)]
b = 0
for _ in range(wl.prefill):
    lib.twg_synth_stream_device(ctx.handle, wl.nodes, b * B, B, wl.seed, dev[0].data_ptr(), dev[1].data_ptr(), dev[2].data_ptr())
    w.ingest_batch_device(dev[0].data_ptr(), dev[1].data_ptr(), dev[2].data_ptr(), B, stats=False)
    b += 1
hosts = [torch.empty((B, 3), dtype=torch.int64, pin_memory=True) for _ in range(6)]
for i, h in enumerate(hosts):
    lib.twg_synth_stream_host(wl.nodes, (b + i) * B, B, wl.seed, C.c_void_p(h.data_ptr()))
cap = wl.walks * 8
outs = [[torch.empty(wl.walks + 1, dtype=torch.int64, pin_memory=True), torch.empty(cap, dtype=torch.int64, pin_memory=True),
         torch.empty(cap, dtype=torch.int64, pin_memory=True)] for _ in range(2)]
cfg = tw.WalkConfig(walk_length=80, start_mode=tw.StartMode.Sampled, total_walks=wl.walks, bias=tw.BiasKind.ExponentialIndex, seed=5)
pending = [None, None]
lib.twg_stage_batch(ctx.handle, 0, C.c_void_p(hosts[0].data_ptr()), B)
ctx.sync()
for k in range(6):
    t = [time.perf_counter()]
    if mode == "pipe" and k + 1 < 6:
        lib.twg_stage_batch(ctx.handle, (k + 1) % 2, C.c_void_p(hosts[k + 1].data_ptr()), B)
    if mode != "pipe":
        lib.twg_stage_batch(ctx.handle, k % 2, C.c_void_p(hosts[k].data_ptr()), B)
    t.append(time.perf_counter())
    assert lib.twg_window_ingest_staged(w.handle, k % 2, None) == 0
    t.append(time.perf_counter())
    snap = w.snapshot()
    ws = tw.generate_walks(snap, cfg, variant=tw.Variant.FullWalk)
    t.append(time.perf_counter())
    slot = k % 2
    if pending[slot] is not None:
        lib.twg_walkset_wait(pending[slot].handle)
    t.append(time.perf_counter())
    tot = C.c_uint64()
    off, nodes, times = outs[slot]
    assert lib.twg_walkset_download_compact_async(ws.handle, C.c_void_p(off.data_ptr()), C.c_void_p(nodes.data_ptr()),
                                                  C.c_void_p(times.data_ptr()), nodes.numel(), C.byref(tot)) == 0
    if mode != "pipe":
        lib.twg_walkset_wait(ws.handle)
    pending[slot] = ws
    t.append(time.perf_counter())
    d = [1e3 * (t[i + 1] - t[i]) for i in range(len(t) - 1)]
    print(f"step {k}: stage {d[0]:6.1f}  ingest {d[1]:6.1f}  walks {d[2]:6.1f}  wait {d[3]:6.1f}  compact+issue {d[4]:6.1f}  total {1e3*(t[-1]-t[0]):6.1f} ms", flush=True)
