#!/bin/bash
# Same-box A/B of the shared-panel multi-RHS solve step: TMA-fed (libSTMA) vs cp.async (libSCPA)
for it in 1 2; do
  for lib in build/ab/libSTMA.so build/ab/libSCPA.so; do
    cp "$lib" paper_2208_06290_b200/lib/libhodlr_b200.so
    echo "== $lib r=32"; python tools/cfg5_ab.py 16 17 24 32 64 128 256 2>/dev/null
    echo "== $lib r=64 N=2^21"; CFG5_N=2097152 CFG5_R=64 python tools/cfg5_ab.py 25 32 64 128 256 2>/dev/null
  done
done
cp build/ab/libSTMA.so paper_2208_06290_b200/lib/libhodlr_b200.so
