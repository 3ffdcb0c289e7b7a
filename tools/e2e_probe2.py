"""Per-iteration timing of the host->device factorization (dev probe): upload-only vs factorize_from_host."""
import sys, time
sys.path.insert(0, ".")
import torch
import paper_2208_06290_b200 as hb
n, m, r = 1 << 20, 64, 32
h0 = hb.random_hodlr(n, m, r, seed=0, s=1.0)
Dh, Uh, Vh = h0.D.cpu().pin_memory(), h0.U.cpu().pin_memory(), h0.V.cpu().pin_memory()
b = torch.randn(n, dtype=torch.float64).pin_memory()
nb = (Dh.numel() + Uh.numel() + Vh.numel()) * 8
D, U, V = torch.empty_like(h0.D), torch.empty_like(h0.U), torch.empty_like(h0.V)
del h0
for it in range(6):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    D.copy_(Dh, non_blocking=True); U.copy_(Uh, non_blocking=True); V.copy_(Vh, non_blocking=True)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"upload only {1e3 * (t1 - t0):.1f} ms ({nb / (t1 - t0) / 1e9:.1f} GB/s)", flush=True)
del D, U, V
torch.cuda.empty_cache()
for it in range(8):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    f = hb.factorize_from_host(n, m, r, Dh, Uh, Vh, check=False)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    x = hb.solve(f, b)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"factorize_from_host {1e3 * (t1 - t0):.1f} ms ({nb / (t1 - t0) / 1e9:.1f} GB/s)  solve {1e3 * (t2 - t1):.2f} ms  "
          f"mem {torch.cuda.memory_allocated() / 1e9:.1f} GB reserved {torch.cuda.memory_reserved() / 1e9:.1f}", flush=True)
    del f, x
