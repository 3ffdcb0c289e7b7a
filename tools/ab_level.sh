#!/bin/bash
# Same-box A/B of the level kernel feeds: TMA (level_update5, default) vs cp.async (level_update4).
# Builds: build/ab/libTMA.so, build/ab/libCPA.so.  3 alternating rounds.
for it in 1 2 3; do
  for lib in build/ab/libTMA.so build/ab/libCPA.so; do
    cp "$lib" paper_2208_06290_b200/lib/libhodlr_b200.so
    echo "== $lib"; python tools/phase_time.py 2>/dev/null | sed -n 1,2p
  done
done
cp build/ab/libTMA.so paper_2208_06290_b200/lib/libhodlr_b200.so
