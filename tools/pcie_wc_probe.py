"""H2D bandwidth of 1.2 GB from pinned host memory: default vs write-combined
(cudaHostAllocWriteCombined), alone and with a concurrent 0.7 GB D2H."""
import ctypes
import time

import torch
from cuda.bindings import runtime as rt

n = 1_200_000_000
d = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(700_000_000, dtype=torch.uint8, device="cuda")
err, p_wc = rt.cudaHostAlloc(n, rt.cudaHostAllocWriteCombined)
err2, p_def = rt.cudaHostAlloc(n, rt.cudaHostAllocDefault)
err3, p_out = rt.cudaHostAlloc(700_000_000, rt.cudaHostAllocDefault)
ctypes.memset(p_wc, 1, n)
ctypes.memset(p_def, 1, n)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for name, p in (("default", p_def), ("write-combined", p_wc)):
    for conc in (False, True):
        best = 1e9
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            rt.cudaMemcpyAsync(d.data_ptr(), p, n, rt.cudaMemcpyKind.cudaMemcpyHostToDevice, s1.cuda_stream)
            if conc:
                rt.cudaMemcpyAsync(p_out, d2.data_ptr(), 700_000_000, rt.cudaMemcpyKind.cudaMemcpyDeviceToHost,
                                   s2.cuda_stream)
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        print(f"{name:15s} concurrent_d2h={conc}: {best*1e3:6.2f} ms  H2D {n/best/1e9:5.1f} GB/s")
