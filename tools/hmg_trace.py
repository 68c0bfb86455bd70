"""Per-phase times of the h-multigrid coarse CG from the barrier trace of an experiment build
(PMG_LIB=.../libpmg_trace.so, built with -DPMG_HMG_TRACE).  python tools/hmg_trace.py [p]"""
import sys, os, ctypes, collections
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np
import torch
import paper_1808_03595_b200 as pmg, pmg_inputs as pi
lib = ctypes.CDLL(os.environ["PMG_LIB"])
p = int(sys.argv[1]) if len(sys.argv) > 1 else 2
case = pi.config(int(sys.argv[2]) if len(sys.argv) > 2 else 3, p=p) if len(sys.argv) <= 2 or sys.argv[2] == "3" else pi.config(int(sys.argv[2]))
s = pmg.Solver(case.k, case.widths, case.p, case.lam)
L = s.nlevels - 1
x = [s.grid_coords(L, d) for d in range(3)]
F = s.new_grid(); s.weak_rhs(torch.from_numpy(case.f_nodal(x)).cuda(), F)
u = s.new_grid()
for rep_ in range(2):
    buf = (ctypes.c_ulonglong * (2 * 8192))()
    lib.pmg_debug_hmg_trace(buf, 8192)
    rep = s.solve(F, u, 1e-10)
    torch.cuda.synchronize()
    n = lib.pmg_debug_hmg_trace(buf, 8192)
a = np.array(buf[:2 * n], dtype=np.int64).reshape(-1, 2)
dt = np.diff(a[:, 0]) / 1e3
tags = a[1:, 1]
acc = collections.defaultdict(list)
for t, d in zip(tags, dt):
    acc[int(t)].append(d)
print("barriers", n, "total us", (a[-1, 0] - a[0, 0]) / 1e3, "cycles", rep["cycles"], "coarse its", rep.get("coarse_iters"))
names = {12: "restrict-x1", 13: "restrict-x2", 1: "pre-sweep", 2: "residual", 3: "restrict", 4: "coarsest", 5: "prolong", 6: "post1", 7: "post2",
         8: "r.z (L=0)", 9: "init", 10: "apply+p.q", 11: "x,r update"}
for t in sorted(acc):
    v = acc[t]
    print(f"tag {t:4d} {names.get(t % 100, '?'):12s} level {t // 100}: n={len(v):4d} mean {np.mean(v):9.2f} us  sum {np.sum(v):10.1f} us")
