"""profiles/traffic.json from an ncu --csv capture of the level-step launches
(-k regex:level_update: level_update6 plus the level_update4/5 remainder and
small-level launches; dram__bytes_read.sum + dram__bytes_write.sum per launch,
one factorize+solve per iteration of tools/profile_once.py; the second
iteration is used).  usage: traffic_json.py capture.csv [level_steps=13]"""
import csv, json, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ii, mi, vi, ui = h.index("ID"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
per = collections.OrderedDict()
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3}
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    d = per.setdefault(int(r[ii]), {})
    d[r[mi]] = float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
launches = list(per.values())
launches = launches[len(launches) // 2:]  # second (warm) factorize
out = {
    "kernel": "level phase: level_update6_kernel + level_update4/5 (remainder groups, small levels)",
    "source": sys.argv[1].split("/")[-1],
    "levels": [{"dram_bytes": l["dram__bytes_read.sum"] + l["dram__bytes_write.sum"],
                "read": l["dram__bytes_read.sum"], "write": l["dram__bytes_write.sum"],
                "ms": l["gpu__time_duration.sum"] * 1e3} for l in launches],
}
tot = sum(l["dram_bytes"] for l in out["levels"])
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 13
out["launches"] = len(out["levels"])
out["level_steps"] = steps
out["bytes_per_level_step"] = tot / steps
out["level_update_bytes_per_launch"] = tot / steps  # key read by bench.py: per level step (all launches of a level)
out["total_dram_bytes_per_step"] = tot
print(json.dumps(out, indent=1))
