#!/bin/bash
# Round-2 ncu evidence (one GPU): launch list of one factorize+solve, and --set full
# captures of the dominant level kernel at levels 13, 7 and 1 (second iteration of
# tools/profile_once.py: 13 level launches per factorization), the K apply at level 13,
# the small-batch window LU and the solve level kernel.
mkdir -p gpurun_out
T=${TAG:-r02}
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv python tools/profile_once.py > /dev/null 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:level_update[45] --csv --log-file gpurun_out/${T}_level_traffic.csv python tools/profile_once.py > /dev/null 2>&1
for spec in "13:13" "7:19" "1:25"; do
  lv=${spec%%:*}; skip=${spec##*:}
  ncu --set full --clock-control none --import-source on -k regex:level_update[45] --launch-skip $skip -c 1 -o gpurun_out/${T}_level4_l${lv} -f python tools/profile_once.py > /dev/null 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:tri_apply2 --launch-skip 15 -c 1 -o gpurun_out/${T}_kapply_l13 -f python tools/profile_once.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:getrf_win --launch-skip 20 -c 1 -o gpurun_out/${T}_getrf_win -f python tools/profile_once.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:solve_level --launch-skip 16 -c 1 -o gpurun_out/${T}_solve_level -f python tools/profile_once.py > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/${T}_launches.csv > gpurun_out/${T}_launch_summary.txt 2>&1
python tools/launch_list.py gpurun_out/${T}_launches.csv > gpurun_out/${T}_launch_list.txt 2>&1
python tools/traffic_json.py gpurun_out/${T}_level_traffic.csv > gpurun_out/${T}_traffic.json 2>&1
python tools/ncu_summary.py gpurun_out/${T}_level4_l13.ncu-rep gpurun_out/${T}_level4_l7.ncu-rep gpurun_out/${T}_level4_l1.ncu-rep gpurun_out/${T}_kapply_l13.ncu-rep gpurun_out/${T}_getrf_win.ncu-rep gpurun_out/${T}_solve_level.ncu-rep > gpurun_out/${T}_ncu_summary.txt 2>&1
echo done
