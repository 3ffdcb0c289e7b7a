#!/bin/bash
# compute-sanitizer evidence (round 2): memcheck, racecheck and synccheck of
# tools/sanitize_small.py (every fused kernel family at small sizes).
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 python tools/sanitize_small.py \
    > gpurun_out/sanitize_${tool}.txt 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/sanitize_${tool}.txt
done
