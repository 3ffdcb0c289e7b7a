#!/bin/bash
# TMA level kernel: launch list + level-13 / level-1 captures (round 2, after the A/B)
mkdir -p gpurun_out
T=${TAG:-r02b}
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv python tools/profile_once.py > /dev/null 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:level_update --csv --log-file gpurun_out/${T}_level_traffic.csv python tools/profile_once.py > /dev/null 2>&1
for spec in "13:13" "7:19" "1:25"; do
  lv=${spec%%:*}; skip=${spec##*:}
  ncu --set full --clock-control none --import-source on -k regex:level_update --launch-skip $skip -c 1 -o gpurun_out/${T}_level_l${lv} -f python tools/profile_once.py > /dev/null 2>&1
done
python tools/launch_list.py gpurun_out/${T}_launches.csv > gpurun_out/${T}_launch_list.txt 2>&1
python tools/launch_summary.py gpurun_out/${T}_launches.csv > gpurun_out/${T}_launch_summary.txt 2>&1
python tools/traffic_json.py gpurun_out/${T}_level_traffic.csv > gpurun_out/${T}_traffic.json 2>&1
python tools/ncu_summary.py gpurun_out/${T}_level_l13.ncu-rep gpurun_out/${T}_level_l7.ncu-rep gpurun_out/${T}_level_l1.ncu-rep > gpurun_out/${T}_ncu_summary.txt 2>&1
echo done
