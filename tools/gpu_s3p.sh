mkdir -p gpurun_out
cp build/ab/libPIPE.so paper_2208_06290_b200/lib/libhodlr_b200.so
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/s3p_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/s3p_pytest.log; grep -E "FAIL|Error|assert" gpurun_out/s3p_pytest.log | head
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s3p_launches.csv python tools/profile_once.py > /dev/null 2>&1
python tools/launch_list.py gpurun_out/s3p_launches.csv > gpurun_out/s3p_launch_list.txt 2>&1
head -8 gpurun_out/s3p_launch_list.txt
# (A/B of the rejected pipelined leaf kernel; libraries no longer built)
# bash tools/ab_libs2.sh build/ab/libPIPE.so build/ab/libNOPIPE.so > gpurun_out/s3p_ab.txt 2>&1
cut -c1-330 gpurun_out/s3p_ab.txt
