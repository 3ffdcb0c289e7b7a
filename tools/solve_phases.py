"""Solve phase breakdown (leaf / K / level, CUDA events) per nrhs (dev tool).
usage: python tools/solve_phases.py N R nrhs...   (eager launches)"""
import sys, ctypes as C
sys.path.insert(0, ".")
import torch
import paper_2208_06290_b200 as hb
from paper_2208_06290_b200 import _lib
n, r = int(sys.argv[1]), int(sys.argv[2])
lib = _lib.load()
f = hb.factorize(hb.random_hodlr(n, 64, r, seed=0, s=1.0), check=False)
for nrhs in [int(x) for x in sys.argv[3:]]:
    B = torch.randn(n, nrhs, dtype=torch.float64, device="cuda")
    for _ in range(2):
        hb.solve(f, B, graph=False)
    torch.cuda.synchronize()
    best = None
    for _ in range(3):
        lib.hodlr_profile_enable(1)
        hb.solve(f, B, graph=False); torch.cuda.synchronize()
        ph = (C.c_double * 9)(); lib.hodlr_profile_read(ph, 9); lib.hodlr_profile_enable(0)
        v = [round(ph[i], 3) for i in (5, 6, 7, 8)]
        if best is None or sum(v) < sum(best):
            best = v
    print(f"nrhs={nrhs} gemm={best[0]} leaf={best[1]} k={best[2]} level={best[3]} total={sum(best):.3f}", flush=True)
