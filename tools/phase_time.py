"""Factor/solve times + per-phase breakdown at cfg2 (dev tool; bench.py is the contract)."""
import sys, ctypes as C
sys.path.insert(0, ".")
import torch
import paper_2208_06290_b200 as hb
from paper_2208_06290_b200 import _lib

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
r = int(sys.argv[2]) if len(sys.argv) > 2 else 32
s = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
lib = _lib.load()
h0 = hb.random_hodlr(n, 64, r, seed=0, s=s)
hw = h0.clone()
b = torch.randn(n, dtype=torch.float64, device="cuda")
def run(k):
    out = []
    for _ in range(k):
        hw.D.copy_(h0.D); hw.U.copy_(h0.U)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record(); f = hb.factorize(hw, check=False); e[1].record(); x = hb.solve(f, b, graph=False); e[2].record()
        out.append(e)
    torch.cuda.synchronize()
    return [round(e[0].elapsed_time(e[1]), 3) for e in out], [round(e[1].elapsed_time(e[2]), 3) for e in out], x
run(2)
tf, ts, x = run(5)
print("factor ms", tf, "solve ms", ts)
lib.hodlr_profile_enable(1); run(1)
ph = (C.c_double * 9)(); lib.hodlr_profile_read(ph, 9); lib.hodlr_profile_enable(0)
print({k: round(ph[i], 3) for i, k in enumerate(_lib.PHASES)})
print("relres", float(torch.linalg.norm(h0.matvec(x) - b) / torch.linalg.norm(b)))
