"""cfg5 multi-RHS solve times for a list of nrhs (dev timing tool)."""
import os, statistics, sys
sys.path.insert(0, ".")
import torch
import paper_2208_06290_b200 as hb
n, m, r = int(os.environ.get("CFG5_N", 1 << 20)), 64, int(os.environ.get("CFG5_R", 32))
f = hb.factorize(hb.random_hodlr(n, m, r, seed=0, s=1.0), check=False)
out = []
for nrhs in [int(x) for x in sys.argv[1:]]:
    B = torch.randn(n, nrhs, dtype=torch.float64, device="cuda")
    ts = []
    for it in range(5):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); hb.solve(f, B); e1.record(); torch.cuda.synchronize()
        if it >= 2:
            ts.append(e0.elapsed_time(e1))
    out.append(f"{nrhs}:{statistics.median(ts):.2f}")
print(" ".join(out))
