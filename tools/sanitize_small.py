"""Small factorize + solve + matvec + build through every fused kernel family
(fp64 r = 16 / 32 / 64, fp32 r = 8, multi-RHS, window LU, graph replay) -- the
workload of the compute-sanitizer runs (tools/sanitize.sh)."""
import sys
sys.path.insert(0, ".")
import torch
import paper_2208_06290_b200 as hb

torch.manual_seed(0)
for n, m, r, dt in ((1 << 12, 64, 32, torch.float64), (1 << 11, 32, 16, torch.float64),
                    (1 << 12, 64, 64, torch.float64), (1 << 12, 64, 8, torch.float32)):
    h = hb.random_hodlr(n, m, r, seed=1, s=4.0, dtype=dt)
    f = hb.factorize(h.clone())
    for nrhs in (1, 3, 20):
        b = torch.randn(n, nrhs, dtype=dt, device="cuda")
        x = hb.solve(f, b, graph=False)
        y = h.matvec(x)
    print(n, m, r, dt, float(torch.linalg.norm(y - b) / torch.linalg.norm(b)))
hl = hb.laplace_dl_hodlr(1 << 12, 64, 16)
print("laplace build ok", float(hl.U.abs().max()))
torch.cuda.synchronize()
