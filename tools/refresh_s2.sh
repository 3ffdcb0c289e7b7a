#!/bin/bash
# Round-2 (session 2) measurement refresh in one GPU call: bench line, cfg1/cfg4/cfg5
# configs, cfg5 at N=2^22 r=64, cfg3 full size.
mkdir -p gpurun_out
T=${TAG:-s2}
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"; cat gpurun_out/${T}_bench.json | head -c 600; echo
timeout 900 python tools/bench_configs.py cfg1 cfg5 > gpurun_out/${T}_configs.jsonl 2>&1; echo "configs rc=$?"; tail -3 gpurun_out/${T}_configs.jsonl
timeout 900 python tools/cfg5_full.py > gpurun_out/${T}_cfg5_full.jsonl 2>&1; echo "cfg5 rc=$?"; cat gpurun_out/${T}_cfg5_full.jsonl
timeout 1200 python tools/cfg3_full.py --gaussian > gpurun_out/${T}_cfg3_full.txt 2>&1; echo "cfg3 rc=$?"; tail -3 gpurun_out/${T}_cfg3_full.txt
