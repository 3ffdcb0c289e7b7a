#!/bin/bash
# launch list (per-kernel durations + DRAM bytes) of one cfg2 matvec: bash tools/matvec_ncu.sh [nrhs]
mkdir -p gpurun_out
NRHS=${1:-1}
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/matvec_launches_$NRHS.csv python -c "
import sys; sys.path.insert(0, '.')
import tools.matvec_bench as mb, torch
mb.run(1 << 20, 64, 32, torch.float64, $NRHS, reps=1)
"
python - $NRHS <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(f'gpurun_out/matvec_launches_{sys.argv[1]}.csv')) if len(r) > 10]
hdr = rows[0]; ki = hdr.index('Kernel Name'); mi = hdr.index('Metric Name'); vi = hdr.index('Metric Value')
for r in rows[-9:]:
    if 'matvec' in r[ki]: print(r[ki][:60], r[mi], r[vi])
PY
