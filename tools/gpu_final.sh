#!/bin/bash
# Round-2 final evidence in one GPU call: GPU tests, smoke, the bench line, other
# configs, launch list + level traffic + ncu captures of the level kernels.
mkdir -p gpurun_out
T=${TAG:-r2z}
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${T}_pytest.log
cp gpurun_out/parity_errors.json gpurun_out/${T}_parity_errors.json 2>/dev/null
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"; cat gpurun_out/${T}_bench.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${T}_bench_ref.json 2>&1; tail -1 gpurun_out/${T}_bench_ref.json
timeout 1200 python tools/bench_configs.py cfg1 cfg4 cfg4g > gpurun_out/${T}_configs.jsonl 2>&1; cat gpurun_out/${T}_configs.jsonl
TAG=${T} timeout 1800 bash tools/profile_r02b.sh > /dev/null 2>&1; echo "profile done"
