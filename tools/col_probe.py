"""Per-step timestamps of the column-owner LU (build with -DHODLR_COL_PROBE; dev tool)."""
import sys, ctypes as C
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2208_06290_b200 import _lib
lib = _lib.load()
s = int(sys.argv[1]) if len(sys.argv) > 1 else 64
a = torch.randn(1, s, s, dtype=torch.float64, device="cuda")
sw = torch.empty(1, s, dtype=torch.int32, device="cuda"); pm = torch.empty_like(sw); info = torch.empty(1, dtype=torch.int32, device="cuda")
for _ in range(3):
    b = a.clone()
    lib.hodlr_getrf_batched(0, s, 1, C.c_void_p(b.data_ptr()), s, s * s, C.c_void_p(sw.data_ptr()), C.c_void_p(pm.data_ptr()), C.c_void_p(info.data_ptr()), None, 0, 0, None)
torch.cuda.synchronize()
buf = (C.c_longlong * (128 * 8))()
lib.hodlr_col_probe(buf)
p = np.array(buf, dtype=np.int64).reshape(128, 8)[1:s]
d = np.diff(p[:, :7], axis=1)
print("per-step cycles: wait->upd, upd->keys, keys->argmax, argmax->seed, seed->mult, mult->arrive")
print("median", np.median(d, axis=0), "step period", np.median(np.diff(p[:, 0])))
