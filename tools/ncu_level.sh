#!/bin/bash
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:level_update2 --launch-skip 1 -c 1 -o gpurun_out/level2_l12 -f python tools/profile_once.py > gpurun_out/ncu_l12.log 2>&1; echo rc=$?
ncu --set full --clock-control none --import-source on -k regex:level_update2 --launch-skip 6 -c 1 -o gpurun_out/level2_l7 -f python tools/profile_once.py > gpurun_out/ncu_l7.log 2>&1; echo rc=$?
ncu --set full --clock-control none --import-source on -k regex:tri_apply_kernel --launch-skip 0 -c 2 -o gpurun_out/triapply -f python tools/profile_once.py > gpurun_out/ncu_tri.log 2>&1; echo rc=$?
ncu --set full --clock-control none --import-source on -k regex:getrf_sr --launch-skip 0 -c 2 -o gpurun_out/getrf -f python tools/profile_once.py > gpurun_out/ncu_getrf.log 2>&1; echo rc=$?
