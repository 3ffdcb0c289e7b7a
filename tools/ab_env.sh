#!/bin/bash
# Same-box A/B of environment toggles: bash tools/ab_env.sh "VAR=a" "VAR=b" ...
for cfg in "$@"; do
  for i in 1 2; do
    env $cfg python tools/phase_time.py 2>/dev/null | sed -n 1,2p | python -c "
import sys, ast
l = sys.stdin.read().split('\n')
f = ast.literal_eval(l[0].split('factor ms ')[1].split(' solve')[0])
d = ast.literal_eval(l[1])
print('$cfg', 'factor', min(f), 'level', d['level'])"
  done
done
