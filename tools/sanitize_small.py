"""Small factorize + solve + matvec + build through every fused kernel family
(fp64 r = 16 / 32 / 64, fp32 r = 8, multi-RHS, window LU, graph replay, the
persistent level_update6 with its remainder launches, the staged upload of
pageable host inputs) -- the workload of the compute-sanitizer runs
(tools/sanitize.sh)."""
import sys
sys.path.insert(0, ".")
import torch
import paper_2208_06290_b200 as hb

torch.manual_seed(0)
for n, m, r, dt in ((1 << 12, 64, 32, torch.float64), (1 << 13, 64, 32, torch.float64), (1 << 11, 32, 16, torch.float64),
                    (1 << 12, 64, 64, torch.float64), (1 << 12, 64, 8, torch.float32)):
    h = hb.random_hodlr(n, m, r, seed=1, s=4.0, dtype=dt)
    f = hb.factorize(h.clone())
    for nrhs in (1, 3, 20):
        b = torch.randn(n, nrhs, dtype=dt, device="cuda")
        x = hb.solve(f, b, graph=False)
        y = h.matvec(x)
    print(n, m, r, dt, float(torch.linalg.norm(y - b) / torch.linalg.norm(b)))
h = hb.random_hodlr(1 << 13, 64, 32, seed=2, s=4.0)
fh = hb.factorize_from_host(1 << 13, 64, 32, *(x.cpu().numpy().copy() for x in (h.D, h.U, h.V)))
bh = torch.randn(1 << 13, dtype=torch.float64, device="cuda")
print("from_host (pageable) ok", float(torch.linalg.norm(h.matvec(hb.solve(fh, bh)) - bh) / torch.linalg.norm(bh)))
hl = hb.laplace_dl_hodlr(1 << 12, 64, 16)
print("laplace build ok", float(hl.U.abs().max()))
torch.cuda.synchronize()
