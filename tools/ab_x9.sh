#!/bin/bash
# rank-64 multi-RHS crossover: streaming kernel (9-24 RHS) vs the TMA shared-panel kernel from 9 RHS
for it in 1 2; do
  for lib in build/ab/libRS.so build/ab/libX9.so; do
    cp "$lib" paper_2208_06290_b200/lib/libhodlr_b200.so
    echo "== $lib r=64 N=2^21"; CFG5_N=2097152 CFG5_R=64 python tools/cfg5_ab.py 9 12 16 20 24 2>/dev/null
  done
done
cp build/ab/libRS.so paper_2208_06290_b200/lib/libhodlr_b200.so
