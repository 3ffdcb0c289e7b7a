#!/bin/bash
# cfg4 (fp32, r = 8, N = 2^21) launch list + one full capture of level_f32_kernel at the deepest update level
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cfg4_launches.csv python tools/cfg4_time.py > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows = [r for r in csv.reader(open("gpurun_out/cfg4_launches.csv")) if len(r) > 10]
h = rows[0]; k = h.index("Kernel Name"); v = h.index("Metric Value")
agg = collections.OrderedDict()
for r in rows[1:]:
    n = r[k].split("(")[0][:70]; agg.setdefault(n, [0, 0]); agg[n][0] += 1; agg[n][1] += float(r[v].replace(",", ""))
for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:12]: print(c // 4, round(t / 4e6, 3), "ms/iter", n)
PY
if [ "${FULL:-0}" = 1 ]; then
ncu --set full --clock-control none --import-source on -k regex:getrs_col_kernel --launch-skip 0 -c 1 -o gpurun_out/cfg4_getrs_full -f python tools/cfg4_time.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:level_f32_kernel --launch-skip 1 -c 1 -o gpurun_out/cfg4_levelf32_full -f python tools/cfg4_time.py > /dev/null 2>&1
ncu -i gpurun_out/cfg4_levelf32_full.ncu-rep --page raw --csv | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; v=r[2]
keys=['gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','sm__warps_active.avg.pct_of_peak_sustained_active','launch__registers_per_thread','launch__grid_size','sm__throughput.avg.pct_of_peak_sustained_elapsed','gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed','l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum','smsp__inst_executed.sum','launch__occupancy_limit_registers','smsp__average_warp_latency_issue_stalled_long_scoreboard','smsp__pcsamp_warps_issue_stalled_long_scoreboard','smsp__pcsamp_warps_issue_stalled_lg_throttle','smsp__pcsamp_warps_issue_stalled_barrier','smsp__pcsamp_warps_issue_stalled_membar','smsp__pcsamp_warps_issue_stalled_short_scoreboard','smsp__pcsamp_warps_issue_stalled_wait','smsp__pcsamp_warps_issue_stalled_math_pipe_throttle','smsp__pcsamp_warps_issue_stalled_mio_throttle','smsp__pcsamp_warps_issue_stalled_selected','smsp__pcsamp_warps_issue_stalled_not_selected','smsp__pcsamp_warps_issue_stalled_no_instructions','smsp__pcsamp_warps_issue_stalled_drain']
for k in keys:
    if k in h: print(k, v[h.index(k)])
"
fi
