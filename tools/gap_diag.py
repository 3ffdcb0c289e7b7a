"""Diagnose step-time variation: factorize timed with/without the NVML sampler, with/without restore."""
import sys, time, threading
sys.path.insert(0, ".")
import torch
import paper_2208_06290_b200 as hb
from paper_2208_06290_b200 import _lib
import bench

n = 1 << 20
h0 = hb.random_hodlr(n, 64, 32, seed=0, s=4.0)
hw = h0.clone()
b = torch.randn(n, dtype=torch.float64, device="cuda")
lib = _lib.load()

def run(k, restore=True, prof=False):
    evs = []
    for _ in range(k):
        if restore:
            hw.D.copy_(h0.D); hw.U.copy_(h0.U)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record()
        f = hb.factorize(hw, check=False)
        e[1].record()
        x = hb.solve(f, b)
        e[2].record()
        evs.append(e)
    torch.cuda.synchronize()
    return [round(e[0].elapsed_time(e[1]), 2) for e in evs], [round(e[1].elapsed_time(e[2]), 2) for e in evs]

run(3)
print("plain      ", run(6))
with bench.ClockSampler(0) as c:
    print("sampler    ", run(6))
print("no-restore ", run(6, restore=False))
lib.hodlr_profile_enable(1)
print("profiled   ", run(3))
import ctypes as C
ph = (C.c_double * 9)(); lib.hodlr_profile_read(ph, 9); print([round(v / 3, 2) for v in ph])
lib.hodlr_profile_enable(0)
# host-side time of one factorize call
torch.cuda.synchronize(); t0 = time.perf_counter(); f = hb.factorize(hw, check=False); t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
print("host enqueue ms", (t1 - t0) * 1e3, "total", (t2 - t0) * 1e3)
