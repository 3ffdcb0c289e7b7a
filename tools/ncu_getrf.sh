#!/bin/bash
# ncu --set full (source-level) of the leaf getrf_reg_kernel<64> launch (16384 blocks) of a cfg2-shaped factorization
mkdir -p gpurun_out
T=${TAG:-lu}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:getrf_reg_kernel -c 1 -o gpurun_out/${T}_getrf -f python tools/profile_once.py > gpurun_out/${T}_getrf.log 2>&1
python tools/ncu_summary.py gpurun_out/${T}_getrf.ncu-rep > gpurun_out/${T}_getrf_summary.txt 2>&1
head -5 gpurun_out/${T}_getrf_summary.txt | cut -c1-400
