"""Time the device assembly of the cfg2 operator (Laplace DL, N = 2^20, leaf 64, rank 32) and its factor+solve."""
import sys, time
sys.path.insert(0, ".")
import torch
import paper_2208_06290_b200 as hb
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
for it in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    h = hb.laplace_dl_hodlr(n, 64, 32)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"build N={n}: {1e3 * (t1 - t0):.1f} ms", flush=True)
b = torch.randn(n, dtype=torch.float64, device="cuda")
for it in range(3):
    hh = h.clone(); torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record(); f = hb.factorize(hh); e[1].record(); x = hb.solve(f, b); e[2].record(); torch.cuda.synchronize()
    print(f"factor {e[0].elapsed_time(e[1]):.2f} ms solve {e[1].elapsed_time(e[2]):.2f} ms relres "
          f"{float(torch.linalg.norm(h.matvec(x) - b) / torch.linalg.norm(b)):.2e}", flush=True)
    del f, hh
