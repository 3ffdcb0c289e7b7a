"""Host-side enqueue cost of factorize_from_host, per step (dev probe)."""
import sys, time, cProfile, pstats, io
sys.path.insert(0, ".")
import torch
import paper_2208_06290_b200 as hb
n, m, r = 1 << 20, 64, 32
h0 = hb.random_hodlr(n, m, r, seed=0, s=1.0)
Dh, Uh, Vh = h0.D.cpu().pin_memory(), h0.U.cpu().pin_memory(), h0.V.cpu().pin_memory()
del h0
torch.cuda.empty_cache()
for it in range(7):
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    t0 = time.perf_counter()
    pr.enable()
    f = hb.factorize_from_host(n, m, r, Dh, Uh, Vh, check=False)
    pr.disable()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"it {it}: enqueue {1e3 * (t1 - t0):.1f} ms", flush=True)
    if it in (3, 4):
        s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(8); print(s.getvalue()[:2500])
    del f
