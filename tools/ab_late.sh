#!/bin/bash
# A/B on the same box: LATE (C added after the update products) vs accumulate-from-C for 1-2 groups per warp
set -e
run() { for i in 1 2; do python tools/phase_time.py 2>/dev/null | sed -n 2p | python -c "import sys,ast; d=ast.literal_eval(sys.stdin.read()); print('$1', 'level', d['level'])"; done; }
run A_late
make -j16 NVFLAGS_EXTRA=-DLEVEL4_LATE=0 > /dev/null 2>&1 || true
touch paper_2208_06290_b200/csrc/level.cu
make -j16 NVFLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude -DLEVEL4_LATE=0" > /dev/null 2>&1
run B_nolate
touch paper_2208_06290_b200/csrc/level.cu
make -j16 > /dev/null 2>&1
run A_again
