"""Summarise an ncu --csv launch list: time per kernel name (share of total)."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hdr_i + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0][:90]
    v = float(r[vi].replace(",", ""))
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v[1] for v in agg.values())
unit = "ns"
for k, (c, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{v/1e6:10.3f} ms {100*v/tot:5.1f}%  x{c:<5d} {k}")
print(f"{tot/1e6:10.3f} ms total")
