import time, torch
x = torch.empty(150_000_000, dtype=torch.int64, pin_memory=True)  # 1.2 GB
y = torch.empty(90_000_000, dtype=torch.int64, pin_memory=True)   # 0.72 GB
dx = torch.empty_like(x, device="cuda"); dy = torch.empty_like(y, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2):
    torch.cuda.synchronize(); t = time.perf_counter(); dx.copy_(x, non_blocking=True); torch.cuda.synchronize(); h2d = time.perf_counter() - t
    t = time.perf_counter(); y.copy_(dy, non_blocking=True); torch.cuda.synchronize(); d2h = time.perf_counter() - t
    t = time.perf_counter()
    with torch.cuda.stream(s1): dx.copy_(x, non_blocking=True)
    with torch.cuda.stream(s2): y.copy_(dy, non_blocking=True)
    torch.cuda.synchronize(); both = time.perf_counter() - t
    print(f"H2D 1.2GB {h2d*1e3:.1f} ms ({1.2/h2d:.1f} GB/s)  D2H 0.72GB {d2h*1e3:.1f} ms ({0.72/d2h:.1f} GB/s)  concurrent {both*1e3:.1f} ms")
