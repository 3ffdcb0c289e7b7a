"""Phase breakdown for any (n, r, dtype) (dev tool)."""
import sys, ctypes as C
sys.path.insert(0, ".")
import torch
import paper_2208_06290_b200 as hb
from paper_2208_06290_b200 import _lib
n, r = int(sys.argv[1]), int(sys.argv[2])
dt = torch.float32 if (len(sys.argv) > 3 and sys.argv[3] == "f32") else torch.float64
lib = _lib.load()
h0 = hb.random_hodlr(n, 64, r, seed=0, s=1.0, dtype=dt)
b = torch.randn(n, dtype=dt, device="cuda")
for _ in range(2):
    f = hb.factorize(h0.clone(), check=False); x = hb.solve(f, b)
torch.cuda.synchronize()
h = h0.clone()
lib.hodlr_profile_enable(1)
f = hb.factorize(h, check=False); x = hb.solve(f, b); torch.cuda.synchronize()
ph = (C.c_double * 9)(); lib.hodlr_profile_read(ph, 9); lib.hodlr_profile_enable(0)
print({k: round(ph[i], 3) for i, k in enumerate(_lib.PHASES)})
