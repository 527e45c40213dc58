import time, numpy as np, torch, os
n = 50_000_000
a = torch.empty((n, 3), dtype=torch.int64, pin_memory=True)
a.random_(0, 1 << 40)
b = torch.empty((n, 3), dtype=torch.int32, pin_memory=True)
torch.set_num_threads(os.cpu_count())
print("cpus", os.cpu_count(), "torch threads", torch.get_num_threads())
for _ in range(3):
    t0 = time.perf_counter(); b.copy_(a); dt = time.perf_counter() - t0
    print(f"i64->i32 convert copy: {dt*1e3:.1f} ms  ({(a.numel()*8 + b.numel()*4)/dt/1e9:.1f} GB/s)")
d = torch.empty((n, 3), dtype=torch.int64, device="cuda")
for _ in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter(); d.copy_(a, non_blocking=True); torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(f"H2D pinned 1.2GB: {dt*1e3:.1f} ms ({a.numel()*8/dt/1e9:.1f} GB/s)")
