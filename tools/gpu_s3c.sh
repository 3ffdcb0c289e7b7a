mkdir -p gpurun_out
T=s3c
for spec in "13:0" "7:6"; do
  lv=${spec%%:*}; skip=${spec##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:level_update --launch-skip $skip -c 1 -o gpurun_out/${T}_level_l${lv} -f python tools/profile_once.py > gpurun_out/${T}_ncu_l${lv}.log 2>&1
done
echo done
