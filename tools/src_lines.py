"""Per-CUDA-line stall samples and shared-memory wavefronts from an ncu cuda,sass source page.

    ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > X.csv
    python tools/src_lines.py X.csv [ranges: a-b:name ...]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hi]
si = h.index("Warp Stall Sampling (All Samples)")
wf, wfi = h.index("L1 Wavefronts Shared"), h.index("L1 Wavefronts Shared Ideal")
ie = h.index("Instructions Executed")
data = [r for r in rows[hi + 1:] if len(r) > si and r[0].isdigit() and r[2] == "-"]
f = lambda x: float(x) if x not in ("", "-") else 0.0
tot = sum(f(r[si]) for r in data)
for spec in sys.argv[2:]:
    ab, n = spec.split(":")
    a, b = map(int, ab.split("-"))
    sel = [r for r in data if a <= int(r[0]) <= b]
    print("%-8s samples %5.1f%%  instr %.3g  shared wf %.3g (ideal %.3g)" % (
        n, 100 * sum(f(r[si]) for r in sel) / tot, sum(f(r[ie]) for r in sel),
        sum(f(r[wf]) for r in sel), sum(f(r[wfi]) for r in sel)))
for r in sorted(data, key=lambda r: -f(r[si]))[:30]:
    print("%5s %5.1f%%  wf %8.3g / %8.3g  %s" % (r[0], 100 * f(r[si]) / tot, f(r[wf]), f(r[wfi]), r[1].strip()[:100]))
