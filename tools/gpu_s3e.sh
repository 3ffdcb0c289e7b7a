mkdir -p gpurun_out
cp build/ab/libL6.so paper_2208_06290_b200/lib/libhodlr_b200.so
T=s3e
for spec in "13:0" "7:6"; do
  lv=${spec%%:*}; skip=${spec##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:level_update --launch-skip $skip -c 1 -o gpurun_out/${T}_level_l${lv} -f python tools/profile_once.py > gpurun_out/${T}_ncu_l${lv}.log 2>&1
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv python tools/profile_once.py > /dev/null 2>&1
python tools/launch_list.py gpurun_out/${T}_launches.csv > gpurun_out/${T}_launch_list.txt 2>&1
echo done
