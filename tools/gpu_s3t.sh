mkdir -p gpurun_out
L=L7
cp build/ab/lib$L.so paper_2208_06290_b200/lib/libhodlr_b200.so
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/s3t_pytest_$L.log 2>&1; echo "$L pytest rc=$?"; tail -1 gpurun_out/s3t_pytest_$L.log; grep -E "FAIL|Error|assert" gpurun_out/s3t_pytest_$L.log | head -5
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s3t_launches_$L.csv python tools/profile_once.py > /dev/null 2>&1
python tools/launch_list.py gpurun_out/s3t_launches_$L.csv > gpurun_out/s3t_launch_list_$L.txt 2>&1
grep -E "level_update|level_reduce" gpurun_out/s3t_launch_list_$L.txt | head -24
bash tools/ab_libs2.sh build/ab/libL7.so build/ab/libL6g.so > gpurun_out/s3t_ab.txt 2>&1
cut -c1-300 gpurun_out/s3t_ab.txt
