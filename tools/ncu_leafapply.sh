#!/bin/bash
# ncu --set full (source-level) of the leaf apply tri_apply2_kernel<64,32> and the level-13 K apply tri_apply2_kernel<64,0>
mkdir -p gpurun_out
T=${TAG:-la}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tri_apply2_kernel -c 2 -o gpurun_out/${T}_apply -f python tools/profile_once.py > gpurun_out/${T}_apply.log 2>&1
python tools/ncu_summary.py gpurun_out/${T}_apply.ncu-rep > gpurun_out/${T}_apply_summary.txt 2>&1
grep -E "==|Duration|stalls|dmma" gpurun_out/${T}_apply_summary.txt | cut -c1-300
