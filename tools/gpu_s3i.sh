mkdir -p gpurun_out
L=L6e
cp build/ab/lib$L.so paper_2208_06290_b200/lib/libhodlr_b200.so
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_ops.py -q -x > gpurun_out/s3i_pytest_$L.log 2>&1; echo "$L pytest rc=$?"; tail -1 gpurun_out/s3i_pytest_$L.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s3i_launches_$L.csv python tools/profile_once.py > /dev/null 2>&1
python tools/launch_list.py gpurun_out/s3i_launches_$L.csv > gpurun_out/s3i_launch_list_$L.txt 2>&1
grep level_update gpurun_out/s3i_launch_list_$L.txt | head -13
bash tools/ab_libs2.sh build/ab/libL6d.so build/ab/libL6e.so > gpurun_out/s3i_ab.txt 2>&1
cat gpurun_out/s3i_ab.txt | cut -c1-250
