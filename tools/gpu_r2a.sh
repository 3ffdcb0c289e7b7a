set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r2a_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r2a_pytest.log
timeout 300 python tests/golden/make_cfg_golden.py cfg1 > gpurun_out/r2a_cfg1_golden.log 2>&1; echo "golden rc=$?"; tail -3 gpurun_out/r2a_cfg1_golden.log
timeout 300 python -m pytest tests/test_gpu_baseline_ops.py -q > gpurun_out/r2a_baseops.log 2>&1; tail -8 gpurun_out/r2a_baseops.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err; echo "bench rc=$?"; cat gpurun_out/r2a_bench.json; tail -3 gpurun_out/r2a_bench.err
timeout 900 python bench.py --gpus 2 --dist-backend gloo --workload cfg2 --steps 3 --warmup 1 > gpurun_out/r2a_gloo2.json 2> gpurun_out/r2a_gloo2.err; echo "gloo rc=$?"; cat gpurun_out/r2a_gloo2.json; tail -3 gpurun_out/r2a_gloo2.err
