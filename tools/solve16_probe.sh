#!/bin/bash
# 16-RHS solve at cfg2 shape: phase breakdown (eager events), launch list, ncu of one level step.
mkdir -p gpurun_out
T=${TAG:-s16}
timeout 300 python tools/solve_phases.py 1048576 32 1 8 16 24 32 > gpurun_out/${T}_phases.txt 2>&1; cat gpurun_out/${T}_phases.txt
cat > /tmp/s16.py <<'PY'
import sys; sys.path.insert(0, ".")
import torch, paper_2208_06290_b200 as hb
n = 1 << 20
f = hb.factorize(hb.random_hodlr(n, 64, 32, seed=0, s=1.0), check=False)
B = torch.randn(n, 16, dtype=torch.float64, device="cuda")
for _ in range(2):
    hb.solve(f, B, graph=False); torch.cuda.synchronize()
PY
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv python /tmp/s16.py > /dev/null 2>&1
python tools/launch_list.py gpurun_out/${T}_launches.csv > gpurun_out/${T}_launch_list.txt 2>&1
tail -45 gpurun_out/${T}_launch_list.txt
ncu --set full --import-source on --clock-control none -k regex:solve_step -s 16 -c 1 -o gpurun_out/${T}_step -f python /tmp/s16.py > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/${T}_step.ncu-rep > gpurun_out/${T}_step_summary.txt 2>&1; head -8 gpurun_out/${T}_step_summary.txt | cut -c1-400
