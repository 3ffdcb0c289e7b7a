mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/s3q_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/s3q_pytest.log
timeout 300 python tools/cfg5_ab.py 1 8 16 24 32 2>&1 | tail -1
timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 --error-exitcode 9 python tools/sanitize_small.py > gpurun_out/sanitize_racecheck.txt 2>&1; echo "racecheck rc=$?"; tail -3 gpurun_out/sanitize_racecheck.txt
