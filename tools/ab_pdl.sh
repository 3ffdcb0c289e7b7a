#!/bin/bash
# Same-box A/B: programmatic dependent launch on (libPDL) vs off (libNOPDL).
# cfg2 step (graphs) via bench.py without the CPU / e2e legs, cfg1 factor/solve.
mkdir -p gpurun_out
for it in 1 2; do
  for lib in build/ab/libPDL.so build/ab/libNOPDL.so; do
    cp "$lib" paper_2208_06290_b200/lib/libhodlr_b200.so
    echo "== $lib"
    timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('cfg2 step', round(d['ms_per_step'],3), 'factor', round(d['t_factor_ms'],3), 'solve', round(d['t_solve_ms'],3), 'eager', d['eager_ms'], 'level', round(d['phase_ms']['level'],3), 'relres', d['relres'])"
    timeout 600 python tools/bench_configs.py cfg1 2>/dev/null | tail -1 | cut -c1-300
  done
done
cp build/ab/libPDL.so paper_2208_06290_b200/lib/libhodlr_b200.so
