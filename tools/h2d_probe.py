"""Host->device bandwidth from pinned memory: one stream vs two (dev probe)."""
import time, torch
n = 1 << 29  # 4 GiB of fp64
a = torch.empty(n, dtype=torch.float64).pin_memory()
b = torch.empty(n, dtype=torch.float64).pin_memory()
da = torch.empty(n, dtype=torch.float64, device="cuda"); db = torch.empty_like(da)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for it in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    with torch.cuda.stream(s1):
        da.copy_(a, non_blocking=True); db.copy_(b, non_blocking=True)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    with torch.cuda.stream(s1):
        da.copy_(a, non_blocking=True)
    with torch.cuda.stream(s2):
        db.copy_(b, non_blocking=True)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"one stream {2 * 8 * n / (t1 - t0) / 1e9:.1f} GB/s   two streams {2 * 8 * n / (t2 - t1) / 1e9:.1f} GB/s")
