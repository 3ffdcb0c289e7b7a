#!/bin/bash
# same-box A/B of level_f32 row-loop unroll (dev experiment)
run() { for i in 1 2; do python tools/cfg4_time.py 2>/dev/null | tail -2 | head -1 | sed "s/^/$1 /"; done; }
run A_unroll2
sed -i 's/^#pragma unroll 2$/#pragma unroll 1/' paper_2208_06290_b200/csrc/level_f32.cu
make -j16 > /dev/null 2>&1
run B_unroll1
sed -i 's/^#pragma unroll 1$/#pragma unroll 4/' paper_2208_06290_b200/csrc/level_f32.cu
make -j16 > /dev/null 2>&1
run C_unroll4
