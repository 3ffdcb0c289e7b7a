#!/bin/bash
# Same-box A/B of multi-RHS solve builds: bash tools/ab_solve_multi.sh build/ab/libA.so build/ab/libB.so ...
for it in 1 2; do
  for lib in "$@"; do
    cp "$lib" paper_2208_06290_b200/lib/libhodlr_b200.so
    echo "== $lib r=32 N=2^20"; python tools/cfg5_ab.py 1 8 9 12 16 24 32 48 64 128 2>/dev/null
    echo "== $lib r=64 N=2^21"; CFG5_N=2097152 CFG5_R=64 python tools/cfg5_ab.py 1 8 9 16 24 32 48 64 128 2>/dev/null
  done
done
cp "$1" paper_2208_06290_b200/lib/libhodlr_b200.so
