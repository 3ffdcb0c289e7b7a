"""Key ncu metrics (details page) for every kernel in a .ncu-rep: SOL, pipes, stalls, traffic."""
import csv, subprocess, sys, io, collections
KEYS = ["Duration", "Elapsed Cycles", "DRAM Throughput", "Compute (SM) Throughput", "Memory Throughput",
        "L2 Hit Rate", "Achieved Occupancy", "Registers Per Thread", "Issue Slots Busy", "Grid Size", "Block Size",
        "Dynamic Shared Memory Per Block", "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction",
        "Executed Ipc Active", "Local Memory Spilling Requests"]
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.DictReader(io.StringIO(out)))
    by = collections.OrderedDict()
    for r in rows:
        by.setdefault((r["ID"], r["Kernel Name"][:60]), {})[r["Metric Name"]] = (r["Metric Value"], r["Metric Unit"])
    for (i, k), d in by.items():
        print(f"== {rep} [{i}] {k}")
        print("   " + "; ".join(f"{m}={d[m][0]}{d[m][1]}" for m in KEYS if m in d))
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    hdr, units = rr[0], rr[1]
    for row in rr[2:]:
        d = dict(zip(hdr, row))
        want = [h for h in hdr if h.startswith("smsp__average_warp_latency_issue_stalled") or
                h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]
        st = sorted(((float(d[h].replace(",", "") or 0), h) for h in want), reverse=True)[:8]
        print("   stalls:", ", ".join(f"{h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}={v:.2f}" for v, h in st))
        tensor = [h for h in hdr if ("dmma" in h or "pipe_tensor" in h or "pipe_fp64" in h or "pipe_shared" in h
                                     or "pipe_lsu" in h) and ("pct" in h or h.endswith(".ratio"))]
        for h in tensor:
            v = d[h].replace(",", "")
            if ".avg." in h and "elapsed" not in h and v not in ("", "0") and float(v) != 0.0:
                print(f"   {h} = {d[h]} {units[hdr.index(h)]}")
        for h in ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                  "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "sm__pipe_tensor_op_dmma_cycles_active.avg.pct_of_peak_sustained_active",
                  "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
                  "lts__t_bytes.sum", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"):
            if h in d:
                print(f"   {h} = {d[h]} {units[hdr.index(h)]}")
