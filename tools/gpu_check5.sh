mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/s3r_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/s3r_pytest.log
timeout 300 python tools/cfg5_ab.py 1 8 16 24 32 2>&1 | tail -1
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('step', d['ms_per_step'], 'factor', d['t_factor_ms'], 'solve', d['t_solve_ms'], d['eager_ms'])"
