#!/bin/bash
# Round-end refresh in one GPU call: gpu tests, smoke, bench line, other configs,
# matvec, launch list + ncu captures.  Outputs under gpurun_out/ (TAG prefix).
TAG=${TAG:-r01c}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"; cat gpurun_out/${TAG}_bench.json; tail -3 gpurun_out/${TAG}_bench.err
timeout 900 python tools/bench_configs.py > gpurun_out/${TAG}_configs.jsonl 2>&1; echo "configs rc=$?"; cat gpurun_out/${TAG}_configs.jsonl
timeout 300 python tools/matvec_bench.py > gpurun_out/${TAG}_matvec.jsonl 2>&1; cat gpurun_out/${TAG}_matvec.jsonl
if [ "${NCU:-1}" = "1" ]; then
TAG=$TAG timeout 2400 bash tools/profile_round.sh > gpurun_out/${TAG}_profile.log 2>&1; echo "profile rc=$?"
python tools/launch_summary.py gpurun_out/${TAG}_launches.csv > gpurun_out/${TAG}_launch_summary.txt 2>&1; head -30 gpurun_out/${TAG}_launch_summary.txt
python tools/ncu_summary.py gpurun_out/${TAG}_level4_full.ncu-rep gpurun_out/${TAG}_apply2_full.ncu-rep gpurun_out/${TAG}_solve_full.ncu-rep gpurun_out/${TAG}_getrf_full.ncu-rep > gpurun_out/${TAG}_ncu_summary.txt 2>&1
python tools/traffic_json.py gpurun_out/${TAG}_level_traffic.csv > gpurun_out/${TAG}_traffic.json 2>&1; cat gpurun_out/${TAG}_traffic.json | head -20
fi
