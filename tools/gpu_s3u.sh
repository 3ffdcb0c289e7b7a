mkdir -p gpurun_out
cp build/ab/libL6S.so paper_2208_06290_b200/lib/libhodlr_b200.so
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "multi_rhs or graph" > gpurun_out/s3u_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/s3u_pytest.log; grep -E "FAIL|Error|assert" gpurun_out/s3u_pytest.log | head -5
for it in 1 2; do for L in L6S L6S0; do cp build/ab/lib$L.so paper_2208_06290_b200/lib/libhodlr_b200.so; echo "== $L"; timeout 300 python tools/cfg5_ab.py 1 16 64 128 130 192 256 2>&1 | tail -1; done; done
cp build/ab/libL6S.so paper_2208_06290_b200/lib/libhodlr_b200.so
