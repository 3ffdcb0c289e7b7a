mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/s3n_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/s3n_pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/s3n_bench.json 2> gpurun_out/s3n_bench.err; echo "bench rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/s3n_bench.json')); print(d['ms_per_step'], d['t_factor_ms'], d['t_solve_ms'], d['roofline']['frac'], d['clocks'], d['e2e'])"
tail -3 gpurun_out/s3n_bench.err
