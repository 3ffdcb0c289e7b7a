#!/bin/bash
# Same-box A/B of library builds: bash tools/ab_libs.sh build/ab/libA.so build/ab/libB.so ...
# (3 alternating rounds of tools/phase_time.py; the first library is restored afterwards)
for it in 1 2 3; do
  for lib in "$@"; do
    cp "$lib" paper_2208_06290_b200/lib/libhodlr_b200.so
    echo "== $lib"; python tools/phase_time.py 2>/dev/null | sed -n 1,2p
  done
done
cp "$1" paper_2208_06290_b200/lib/libhodlr_b200.so
