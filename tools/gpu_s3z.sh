mkdir -p gpurun_out
cp build/ab/libCA.so paper_2208_06290_b200/lib/libhodlr_b200.so
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/s3z2_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/s3z2_pytest.log; grep -E "FAIL|Error|assert" gpurun_out/s3z2_pytest.log | head -5
bash tools/ab_libs2.sh build/ab/libCA.so build/ab/libCA0.so > gpurun_out/s3z2_ab.txt 2>&1
cut -c1-300 gpurun_out/s3z2_ab.txt
