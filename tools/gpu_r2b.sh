# round-2 GPU check: tests, smoke, bench, cfg1/cfg4 timings
mkdir -p gpurun_out
T=${TAG:-r2b}
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -40 gpurun_out/${T}_pytest.log | grep -v "^\.\.\."
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"; cat gpurun_out/${T}_bench.json; tail -3 gpurun_out/${T}_bench.err
timeout 900 python tools/bench_configs.py cfg1 cfg4 > gpurun_out/${T}_configs.jsonl 2>&1; cat gpurun_out/${T}_configs.jsonl
