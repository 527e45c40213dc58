"""Diagnostic: time device-resident vs host-buffer ingest back to back."""
import ctypes as C
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
host = torch.empty((B, 3), dtype=torch.int64, pin_memory=True)
b = 0
for i in range(12):
    mode = i % 2
    if mode == 0:
        lib.twg_synth_stream_device(ctx.handle, wl.nodes, b * B, B, wl.seed, dev[0].data_ptr(), dev[1].data_ptr(),
                                    dev[2].data_ptr())
        ctx.sync()
        t0 = time.perf_counter()
        st = w.ingest_batch_device(dev[0].data_ptr(), dev[1].data_ptr(), dev[2].data_ptr(), B, stats=True)
        ctx.sync()
        dt = time.perf_counter() - t0
    else:
        lib.twg_synth_stream_host(wl.nodes, b * B, B, wl.seed, C.c_void_p(host.data_ptr()))
        t0 = time.perf_counter()
        st = w.ingest_batch(host.numpy())
        dt = time.perf_counter() - t0
    print(f"batch {b} {'dev ' if mode == 0 else 'host'} {dt*1000:8.1f} ms  rebuild {st.rebuild_duration*1000:8.1f} ms retained {st.retained}", flush=True)
    b += 1
