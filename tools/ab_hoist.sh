#!/bin/bash
# A/B on the same box: W' hoisting variants of level_update4 (dev experiment)
set -e
run() { for i in 1 2; do python tools/phase_time.py 2>/dev/null | sed -n 2p | python -c "import sys,ast; d=ast.literal_eval(sys.stdin.read()); print('$1', 'level', d['level'])"; done; }
run A_gpw12
sed -i 's/        constexpr bool HOIST = GPW == 1 || (!SOLVE \&\& (GPW <= 2 || R <= 16));/        constexpr bool HOIST = false;/' paper_2208_06290_b200/csrc/level.cu
make -j16 > /dev/null 2>&1
run B_nohoist
sed -i 's/        constexpr bool HOIST = false;/        constexpr bool HOIST = GPW == 1 || (!SOLVE \&\& (GPW <= 2 || R <= 16));/' paper_2208_06290_b200/csrc/level.cu
make -j16 > /dev/null 2>&1
run A_again
