"""One warm-up + one profiled factorize/solve (for ncu launch lists)."""
import sys
sys.path.insert(0, ".")
import torch
import paper_2208_06290_b200 as hb

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
r = int(sys.argv[2]) if len(sys.argv) > 2 else 32
s = float(sys.argv[3]) if len(sys.argv) > 3 else 4.0
h0 = hb.random_hodlr(n, 64, r, seed=0, s=s)
for it in range(2):
    h = h0.clone()
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push(f"iter{it}")
    f = hb.factorize(h, check=False)
    b = torch.randn(n, dtype=torch.float64, device="cuda")
    x = hb.solve(f, b)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
res = h0.matvec(x) - b
print("relres", float(torch.linalg.norm(res) / torch.linalg.norm(b)))
