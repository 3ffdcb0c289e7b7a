"""Quick factor/solve timing at a given N (dev tool; bench.py is the contract)."""
import sys, time, math
sys.path.insert(0, ".")
import torch
import paper_2208_06290_b200 as hb

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
m, r = 64, int(sys.argv[2]) if len(sys.argv) > 2 else 32
reps = 3
h0 = hb.random_hodlr(n, m, r, seed=0, s=16.0)
fl = hb.flop_report(n, m, r)["total"]
for it in range(reps + 1):
    h = h0.clone()
    torch.cuda.synchronize()
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record()
    f = hb.factorize(h, check=False)
    e1.record()
    b = torch.randn(n, dtype=torch.float64, device="cuda")
    e1b = torch.cuda.Event(enable_timing=True); e1b.record()
    x = hb.solve(f, b)
    e2.record()
    torch.cuda.synchronize()
    tf, ts = e0.elapsed_time(e1), e1b.elapsed_time(e2)
    print(f"N={n} r={r} factor {tf:.3f} ms ({fl/tf/1e9:.2f} TFLOP/s)  solve {ts:.3f} ms")
res = hb.HodlrMatrix.matvec(h0, x) - b
print("relres", float(torch.linalg.norm(res) / torch.linalg.norm(b)))
