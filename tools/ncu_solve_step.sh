#!/bin/bash
# ncu --set full of solve-step launches (one 1-RHS and one 16-RHS solve at N=2^20, r=32)
mkdir -p gpurun_out
T=${TAG:-ss}
cat > /tmp/ss.py <<'PY'
import sys; sys.path.insert(0, ".")
import torch, paper_2208_06290_b200 as hb
n = 1 << 20
f = hb.factorize(hb.random_hodlr(n, 64, 32, seed=0, s=1.0), check=False)
for nrhs in (1, 16):
    B = torch.randn(n, nrhs, dtype=torch.float64, device="cuda")
    hb.solve(f, B, graph=False); torch.cuda.synchronize()
PY
ncu --set full --import-source on --clock-control none -k regex:"${KREGEX:-solve_step|solve_level_kernel}" -s ${SKIP:-0} -c ${COUNT:-4} -o gpurun_out/${T} -f python /tmp/ss.py > gpurun_out/${T}.log 2>&1
python tools/ncu_summary.py gpurun_out/${T}.ncu-rep > gpurun_out/${T}_summary.txt 2>&1
tail -5 gpurun_out/${T}.log
