#!/bin/bash
# Same-box A/B of two builds of the library: bash tools/ab_lib.sh build/ab/libA.so build/ab/libB.so ...
for it in 1 2; do
  for lib in "$@"; do
    cp "$lib" paper_2208_06290_b200/lib/libhodlr_b200.so
    python tools/phase_time.py 2>/dev/null | sed -n 1,2p | python -c "
import sys, ast
l = sys.stdin.read().split('\n')
f = ast.literal_eval(l[0].split('factor ms ')[1].split(' solve')[0])
d = ast.literal_eval(l[1])
print('$lib', 'factor', min(f), 'level', d['level'])"
  done
done
