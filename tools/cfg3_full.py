"""cfg3 at its full size on ONE B200: N = 2^22, leaf 64, rank 64, fp64 (~160 GB of
operator + factors + workspace; no restore copy).  Seeded exact-HODLR stand-in
(the Gaussian/Matern 3-D point operator has no device builder yet).  Prints
factor / solve time, TFLOP/s and memory.  ``--gaussian``: the cfg3 operator
(Gaussian kernel on 2^22 kd-ordered 3-D points, assembled on the device)."""
import sys, time
sys.path.insert(0, ".")
import torch
import paper_2208_06290_b200 as hb
n, m, r = 1 << 22, 64, 64
torch.cuda.synchronize()
if "--gaussian" in sys.argv:
    t0 = time.perf_counter()
    h = hb.gaussian_hodlr(n, m, r, dim=3, h=0.1, lam=1.0)
    torch.cuda.synchronize()
    print(f"assembled the 3-D Gaussian operator in {time.perf_counter() - t0:.1f} s (incl. host point generation)")
else:
    h = hb.random_hodlr(n, m, r, seed=0, s=1.0)
b = torch.randn(n, dtype=torch.float64, device="cuda")
# a small warm-up at the same rank (kernel attributes, lazy init)
hw = hb.random_hodlr(1 << 16, m, r, seed=1)
hb.solve(hb.factorize(hw, check=False), torch.randn(1 << 16, dtype=torch.float64, device="cuda"))
del hw
torch.cuda.synchronize()
e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
e[0].record(); f = hb.factorize(h, check=False); e[1].record(); x = hb.solve(f, b); e[2].record()
torch.cuda.synchronize()
tf, ts = e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2])
fl = hb.flop_report(n, m, r)["total"]
print(f"cfg3 full N=2^22 r=64 P=1: factor {tf:.1f} ms ({fl / tf / 1e9:.2f} TFLOP/s) solve {ts:.2f} ms "
      f"peak mem {torch.cuda.max_memory_allocated() / 1e9:.1f} GB", flush=True)
