mkdir -p gpurun_out
for it in 1 2; do for lib in R64 L6g; do cp build/ab/lib$lib.so paper_2208_06290_b200/lib/libhodlr_b200.so; echo "== $lib r=64"; timeout 300 python tools/quick_time.py 1048576 64 2>&1 | tail -2; done; done
cp build/ab/libR64.so paper_2208_06290_b200/lib/libhodlr_b200.so
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "64" 2>&1 | tail -1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s3m_launches_r64.csv python tools/profile_once.py 1048576 64 > /dev/null 2>&1
python tools/launch_list.py gpurun_out/s3m_launches_r64.csv > gpurun_out/s3m_launch_list_r64.txt 2>&1
grep -E "level_update" gpurun_out/s3m_launch_list_r64.txt | head -16
