#!/bin/bash
# flakiness check: the GPU suite three times in a row + a bitwise run-to-run check of the cfg2 factorization
mkdir -p gpurun_out
for i in 1 2 3; do timeout 900 python -m pytest tests -m gpu -q -p no:randomly > gpurun_out/rep_pytest_$i.log 2>&1; echo "run $i rc=$?"; tail -1 gpurun_out/rep_pytest_$i.log; done
cat > /tmp/rr.py <<'PY'
import sys; sys.path.insert(0, ".")
import torch, paper_2208_06290_b200 as hb
h0 = hb.laplace_dl_hodlr(1 << 20, 64, 32)
ref = None
for it in range(5):
    f = hb.factorize(h0.clone(), check=False)
    b = torch.ones(1 << 20, dtype=torch.float64, device="cuda")
    x = hb.solve(f, b)
    cur = (f.Y.clone(), f.K.clone(), f.kswaps.clone(), x.clone())
    if ref is None: ref = cur
    else: print("run", it, "bitwise equal:", all(torch.equal(a, c) for a, c in zip(ref, cur)))
PY
timeout 600 python /tmp/rr.py
