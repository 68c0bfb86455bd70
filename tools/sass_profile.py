"""Aggregate an ncu SASS source page (ncu -i X --page source --csv --print-source sass --kernel-name K)
into stall samples per opcode and per contiguous code region.

    python tools/sass_profile.py sass.csv [nregions]
"""
import csv
import collections
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = []
for r in rows[2:]:
    if r and r[0] == "Kernel Name":
        break
    if len(r) > 3 and r[0].startswith("0x"):
        data.append(r)
si, ni, ei = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
wf, wfi = h.index("L1 Wavefronts Shared"), h.index("L1 Wavefronts Shared Ideal")
tot = sum(float(r[ni] or 0) for r in data)
by_op = collections.Counter()
ex_op = collections.Counter()
stalls = collections.Counter()
shw, shwi = 0.0, 0.0
for r in data:
    op = r[si].strip().split()[0] if r[si].strip() else "?"
    if op.startswith("@"):
        op = r[si].strip().split()[1]
    op = op.split(".")[0]
    by_op[op] += float(r[ni] or 0)
    ex_op[op] += float(r[ei] or 0)
    for c in stall_cols:
        stalls[h[c]] += float(r[c] or 0)
    shw += float(r[wf] or 0)
    shwi += float(r[wfi] or 0)
print("total samples %d, instructions %d, shared wavefronts %.3g (ideal %.3g)" % (tot, sum(ex_op.values()), shw, shwi))
print("stalls:", ", ".join("%s %.1f%%" % (k[6:], 100 * v / tot) for k, v in stalls.most_common(8)))
print("samples by opcode:", ", ".join("%s %.1f%%" % (k, 100 * v / tot) for k, v in by_op.most_common(14)))
print("executed by opcode:", ", ".join("%s %.3g" % (k, v) for k, v in ex_op.most_common(14)))
nreg = int(sys.argv[2]) if len(sys.argv) > 2 else 0
if nreg:
    n = len(data)
    for k in range(nreg):
        seg = data[k * n // nreg:(k + 1) * n // nreg]
        s = sum(float(r[ni] or 0) for r in seg)
        ops = collections.Counter()
        for r in seg:
            op = r[si].strip().split()[0] if r[si].strip() else "?"
            ops[op.split(".")[0]] += float(r[ei] or 0)
        print("region %2d [%s..]: %.1f%% samples, top ops %s" % (k, seg[0][0][-5:], 100 * s / tot,
              ", ".join("%s %.2g" % kv for kv in ops.most_common(5))))
if nreg:
    print("per region: executed instructions and top stalls")
    n = len(data)
    for k in range(nreg):
        seg = data[k * n // nreg:(k + 1) * n // nreg]
        ex = sum(float(r[ei] or 0) for r in seg)
        st = collections.Counter()
        for r in seg:
            for c in stall_cols:
                st[h[c][6:]] += float(r[c] or 0)
        s = sum(st.values()) or 1
        print("region %2d: exec %.3g  stalls %s" % (k, ex, ", ".join("%s %.0f%%" % (a, 100 * b / s) for a, b in st.most_common(4))))
