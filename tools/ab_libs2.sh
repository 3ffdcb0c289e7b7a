#!/bin/bash
# Same-box A/B of library builds (args: build/ab/libX.so ...): cfg2 step through
# bench.py (graphs; no CPU / e2e legs) + the cfg1 factor/solve; 2 alternating rounds.
# The first library is restored at the end.
mkdir -p gpurun_out
for it in 1 2; do
  for lib in "$@"; do
    cp "$lib" paper_2208_06290_b200/lib/libhodlr_b200.so
    echo "== $lib"
    timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('cfg2 step', round(d['ms_per_step'],3), 'factor', round(d['t_factor_ms'],3), 'solve', round(d['t_solve_ms'],3), 'eager', d['eager_ms'], 'phases', {k: round(v,3) for k,v in d['phase_ms'].items()}, 'relres', d['relres'])"
    timeout 600 python tools/bench_configs.py cfg1 2>/dev/null | tail -1 | cut -c1-300
  done
done
cp "$1" paper_2208_06290_b200/lib/libhodlr_b200.so
