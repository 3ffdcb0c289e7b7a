#!/bin/bash
# Profiles committed under profiles/ (one GPU, never under a multi-rank command).
# 1. launch list of one factorize+solve (gpu__time_duration, serialised, cold-ish cache)
# 2. DRAM bytes per launch of the dominant kernel (level_update4) for roofline.traffic
# 3. one --set full capture of the dominant kernel at a deep level (summary only is committed)
set -x
mkdir -p gpurun_out
TAG=${TAG:-r01}
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python tools/profile_once.py > /dev/null 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:level_update4 --csv --log-file gpurun_out/${TAG}_level_traffic.csv python tools/profile_once.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:level_update4 --launch-skip 1 -c 1 -o gpurun_out/${TAG}_level4_full -f python tools/profile_once.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:tri_apply2 --launch-skip 0 -c 1 -o gpurun_out/${TAG}_apply2_full -f python tools/profile_once.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:solve_level --launch-skip 2 -c 1 -o gpurun_out/${TAG}_solve_full -f python tools/profile_once.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:getrf_reg --launch-skip 0 -c 1 -o gpurun_out/${TAG}_getrf_full -f python tools/profile_once.py > /dev/null 2>&1
echo done
