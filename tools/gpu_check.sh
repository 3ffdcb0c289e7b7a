#!/bin/bash
# One GPU call: gpu tests, smoke, bench, ncu launch list, one full ncu capture of the level kernel.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
if [ "${NCU:-1}" = "1" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_once.py > gpurun_out/ncu_ll.log 2>&1; echo "ncu ll rc=$?"
python tools/launch_summary.py gpurun_out/launches.csv > gpurun_out/launch_summary.txt; cat gpurun_out/launch_summary.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:level_update_kernel --launch-skip 14 -c 1 -o gpurun_out/level_full -f python tools/profile_once.py > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
tail -3 gpurun_out/ncu_full.log
fi
