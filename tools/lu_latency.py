"""Batched LU (hodlr_getrf_batched, fp64) time per launch vs batch size (dev tool).
usage: python tools/lu_latency.py S batch..."""
import sys, ctypes as C
sys.path.insert(0, ".")
import torch
from paper_2208_06290_b200 import _lib
lib = _lib.load()
s = int(sys.argv[1])
out = []
for nb in [int(x) for x in sys.argv[2:]]:
    a0 = torch.randn(nb, s, s, dtype=torch.float64, device="cuda")
    a = a0.clone()
    sw = torch.empty(nb, s, dtype=torch.int32, device="cuda")
    pm = torch.empty_like(sw)
    info = torch.empty(nb, dtype=torch.int32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    def go():
        return lib.hodlr_getrf_batched(0, s, nb, C.c_void_p(a.data_ptr()), s, s * s, C.c_void_p(sw.data_ptr()),
                                       C.c_void_p(pm.data_ptr()), C.c_void_p(info.data_ptr()), None, 0, 0, C.c_void_p(st))
    for _ in range(3):
        a.copy_(a0); go()
    ts = []
    for _ in range(10):
        a.copy_(a0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); go(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1000)
    out.append(f"{nb}:{min(ts):.1f}us")
print(f"S={s}", " ".join(out))
