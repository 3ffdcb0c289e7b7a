"""The Laplace double-layer operator at N = 2^22 (the paper's largest fp64 Laplace case), rank 32, one B200."""
import sys, time
sys.path.insert(0, ".")
import torch
import paper_2208_06290_b200 as hb
n, m, r = 1 << 22, 64, 32
torch.cuda.synchronize(); t0 = time.perf_counter()
h = hb.laplace_dl_hodlr(n, m, r)
torch.cuda.synchronize(); tb = time.perf_counter() - t0
b = torch.randn(n, dtype=torch.float64, device="cuda")
hw = hb.random_hodlr(1 << 16, m, r, seed=1)
hb.solve(hb.factorize(hw, check=False), torch.randn(1 << 16, dtype=torch.float64, device="cuda"))
for it in range(2):
    hh = h.clone(); torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record(); f = hb.factorize(hh); e[1].record(); x = hb.solve(f, b); e[2].record(); torch.cuda.synchronize()
    rel = float(torch.linalg.norm(h.matvec(x) - b) / torch.linalg.norm(b))
    print(f"Laplace DL N=2^22 r=32: build {tb:.2f} s  factor {e[0].elapsed_time(e[1]):.1f} ms  solve {e[1].elapsed_time(e[2]):.2f} ms  relres {rel:.2e}", flush=True)
    del f, hh

# fp32, rank 8, N = 2^21: the paper's "low accuracy" Laplace case (assembled in fp64, cast)
n2 = 1 << 21
h64 = hb.laplace_dl_hodlr(n2, 64, 8)
h32 = hb.HodlrMatrix(h64.tree, 8, h64.D.float(), h64.U.float(), h64.V.float())
b2 = torch.randn(n2, dtype=torch.float64, device="cuda")
for it in range(3):
    hh = h32.clone(); torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record(); f = hb.factorize(hh, check=False); e[1].record(); x = hb.solve(f, b2.float()); e[2].record()
    torch.cuda.synchronize()
    rel = float(torch.linalg.norm(h64.matvec(x.double()) - b2) / torch.linalg.norm(b2))
    if it:
        print(f"Laplace DL N=2^21 r=8 fp32: factor {e[0].elapsed_time(e[1]):.2f} ms  solve {e[1].elapsed_time(e[2]):.3f} ms  relres {rel:.2e}", flush=True)
    del f, hh
