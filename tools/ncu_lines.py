"""Per-CUDA-source-line stall samples and executed instructions of one kernel launch from an ncu
report (ncu -i R --page source --csv --print-source cuda,sass), top lines first.

    python tools/ncu_lines.py report.ncu-rep kernel_regex [launch_skip] [top]
"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "--kernel-name",
                      "regex:" + kre, "--launch-skip", skip, "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname = ""
agg = []
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0]:
        continue
    try:
        s = float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        ex = float(r[hdr.index("Instructions Executed")] or 0)
    except (ValueError, IndexError):
        continue
    agg.append((s, ex, fname, r[0], r[1].strip()[:90]))
tot_s = sum(a[0] for a in agg) or 1
tot_e = sum(a[1] for a in agg) or 1
print("samples %d, instructions %.3g" % (tot_s, tot_e))
for s, ex, f, ln, src in sorted(agg, reverse=True)[:top]:
    print("%5.1f%% %5.1f%%  %s:%s  %s" % (100 * s / tot_s, 100 * ex / tot_e, f, ln, src))
