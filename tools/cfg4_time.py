"""cfg4 shape: fp32 rank-8 HODLR (preconditioner), N = 2^21, leaf 64 -- factor/solve timing (dev tool)."""
import sys
sys.path.insert(0, ".")
import torch
import paper_2208_06290_b200 as hb
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 21
r = int(sys.argv[2]) if len(sys.argv) > 2 else 8
h0 = hb.random_hodlr(n, 64, r, seed=0, s=1.0, dtype=torch.float32)
b = torch.randn(n, dtype=torch.float32, device="cuda")
fl = hb.flop_report(n, 64, r)["total"]
for it in range(4):
    h = h0.clone()
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record(); f = hb.factorize(h, check=False); e[1].record(); x = hb.solve(f, b); e[2].record()
    torch.cuda.synchronize()
    tf, ts = e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2])
    print(f"fp32 N={n} r={r}: factor {tf:.3f} ms ({fl / tf / 1e9:.2f} TFLOP/s)  solve {ts:.3f} ms")
res = h0.matvec(x) - b
print("relres", float(torch.linalg.norm(res) / torch.linalg.norm(b)))
