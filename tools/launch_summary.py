"""Per-kernel share of one bench step from an ncu launch list (--metrics gpu__time_duration.sum ... --csv).

    python tools/launch_summary.py launches.csv > profiles/<name>.txt
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h, data = rows[hi], rows[hi + 1:]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
gi, bi = h.index("Grid Size"), h.index("Block Size")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "ms": 1e3,
         "nsecond": 1e-3, "usecond": 1, "msecond": 1e3}
launch = collections.OrderedDict()
for r in data:
    d = launch.setdefault(r[0], {"k": r[ki].split("(")[0], "g": r[gi], "b": r[bi]})
    d[r[mi]] = float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for d in launch.values():
    a = agg[(d["k"], d["g"], d["b"])]
    a[0] += 1
    a[1] += d.get("gpu__time_duration.sum", 0.0)
    a[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
tot = sum(a[1] for a in agg.values())
print("ncu launch list (cold cache, serialised): %d launches, %.1f us total" % (len(launch), tot))
print("%-44s %14s %12s %6s %10s %8s %12s" % ("kernel", "grid", "block", "n", "avg_us", "share", "MB/launch"))
for (k, g, b), a in sorted(agg.items(), key=lambda x: -x[1][1]):
    print("%-44s %14s %12s %6d %10.2f %8.3f %12.3f" % (k[:44], g, b, a[0], a[1] / a[0], a[1] / tot, a[2] / a[0] / 1e6))
