mkdir -p gpurun_out
cp build/ab/libNB6.so paper_2208_06290_b200/lib/libhodlr_b200.so
timeout 900 python -m pytest tests/test_gpu_backend.py tests/test_gpu_parity.py -q -x -k "lu or random or golden" > gpurun_out/s3y_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/s3y_pytest.log; grep -E "FAIL|Error|assert" gpurun_out/s3y_pytest.log | head -5
bash tools/ab_libs2.sh build/ab/libNB6.so build/ab/libNB3.so build/ab/libNB2.so build/ab/libNB0.so > gpurun_out/s3y_ab.txt 2>&1
grep -E "==|cfg2" gpurun_out/s3y_ab.txt | cut -c1-330
