mkdir -p gpurun_out
cp build/ab/libL6.so paper_2208_06290_b200/lib/libhodlr_b200.so
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/s3d_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/s3d_pytest.log
bash tools/ab_libs2.sh build/ab/libL6.so build/ab/libBASE.so > gpurun_out/s3d_ab.txt 2>&1
cat gpurun_out/s3d_ab.txt | cut -c1-300
