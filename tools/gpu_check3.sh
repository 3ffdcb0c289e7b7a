mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "from_host" > gpurun_out/s3o_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s3o_pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/s3o_bench.json 2> gpurun_out/s3o_bench.err; echo "bench rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/s3o_bench.json')); print(d['ms_per_step'], d['e2e']['seconds_per_step'], d['e2e']['pageable'])"
tail -3 gpurun_out/s3o_bench.err
nproc
