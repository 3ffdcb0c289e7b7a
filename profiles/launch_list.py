"""Per-launch listing of the second half of an ncu --csv launch list."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r); h = rows[hi]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
gi = h.index("Grid Size") if "Grid Size" in h else None
L = [(r[ki].split('(')[0].replace('void hodlr::', ''), float(r[vi].replace(',', '')), r[gi] if gi else '')
     for r in rows[hi + 1:] if len(r) > vi and r[mi] == "gpu__time_duration.sum"]
L = [x for x in L if 'at::' not in x[0] and 'internal' not in x[0] and 'gemv' not in x[0]]
half = len(L) // 2 if len(sys.argv) < 3 else 0
for name, t, g in L[half:]:
    print(f"{t/1e3:9.1f} us  {name[:44]:44s} {g}")
