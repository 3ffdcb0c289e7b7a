"""cfg5 at its BASELINE size on ONE B200: multi-RHS solve sweep (1..256 RHS) on
the N = 2^22, rank 64 factorization (seeded exact-HODLR stand-in; --gaussian:
the cfg3 Gaussian operator).  The factorization workspace is released before
the sweep (factors ~90 GB + solve workspace + B/X fit in 180 GB)."""
import statistics, sys, time
sys.path.insert(0, ".")
import torch
import paper_2208_06290_b200 as hb
from paper_2208_06290_b200 import hodlr as hmod

n, m, r = 1 << 22, 64, 64
L = 16
h = hb.gaussian_hodlr(n, m, r, dim=3, h=0.1, lam=1.0) if "--gaussian" in sys.argv else hb.random_hodlr(n, m, r, seed=0)
f = hb.factorize(h, check=False)
del h
hmod._WS_CACHE.clear()
torch.cuda.synchronize()
torch.cuda.empty_cache()
per_rhs_flops = 2 * m * n + 4 * r * n * L + 8 * r * r * ((1 << L) - 1)
fbytes = 8 * (m * n + 2 * n * r * L + 4 * r * r * ((1 << L) - 1))
for nrhs in (1, 2, 4, 8, 16, 32, 64, 128, 256):
    B = torch.randn(n, nrhs, dtype=torch.float64, device="cuda") if nrhs > 1 else torch.randn(n, dtype=torch.float64, device="cuda")
    ts = []
    for it in range(4):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); X = hb.solve(f, B, graph=False); e1.record(); torch.cuda.synchronize()
        if it >= 1:
            ts.append(e0.elapsed_time(e1))
        del X
    t = statistics.median(ts)
    print(f'{{"config": "cfg5 N=2^22 r=64 P=1", "nrhs": {nrhs}, "t_solve_ms": {t:.2f}, '
          f'"solve_tflops": {nrhs * per_rhs_flops / t / 1e9:.2f}, "factor_bytes_GBps": {(fbytes + 16 * n * nrhs) / t / 1e6:.0f}, '
          f'"peak_mem_GB": {torch.cuda.max_memory_allocated() / 1e9:.1f}}}', flush=True)
    del B
    hmod._WS_CACHE.clear()
    torch.cuda.empty_cache()
