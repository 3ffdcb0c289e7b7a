#!/bin/bash
# rank-64 factorization (cfg3 family) at N=2^20: phase breakdown + launch list of the level kernels
mkdir -p gpurun_out
T=${TAG:-r64}
timeout 300 python tools/quick_time.py 1048576 64 2>&1 | tail -2
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv python tools/profile_once.py 1048576 64 > /dev/null 2>&1
python tools/launch_list.py gpurun_out/${T}_launches.csv > gpurun_out/${T}_launch_list.txt 2>&1
python tools/launch_summary.py gpurun_out/${T}_launches.csv > gpurun_out/${T}_launch_summary.txt 2>&1
head -20 gpurun_out/${T}_launch_summary.txt
grep -E "level_update" gpurun_out/${T}_launch_list.txt | head -14
