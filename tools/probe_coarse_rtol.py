"""Coarse-CG tolerance probe: cycles, per-cycle contraction, coarse iterations and solve time per
BASELINE config for a range of coarse_rtol values (reading R11)."""
import sys, os, json
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
import paper_1808_03595_b200 as pmg, pmg_inputs as pi

cases = [pi.config(1), pi.config(2), pi.config(3, p=4), pi.config(3, p=16), pi.config(4)]
for case in cases:
    for rt in (1e-8, 1e-6, 1e-5, 1e-4, 1e-3, 1e-2):
        s = pmg.Solver(case.k, case.widths, case.p, case.lam, coarse_rtol=rt)
        L = s.nlevels - 1
        x = [s.grid_coords(L, d) for d in range(3)]
        F = s.new_grid(); s.weak_rhs(torch.from_numpy(case.f_nodal(x)).cuda(), F)
        u = s.new_grid()
        for _ in range(2): s.solve(F, u, 1e-10)
        ts = []
        for _ in range(5):
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(s.stream); rep = s.solve(F, u, 1e-10); b.record(s.stream); b.synchronize(); ts.append(a.elapsed_time(b))
        h = rep["history"]
        print(json.dumps({"case": case.name, "coarse_rtol": rt, "ms": round(sum(ts) / len(ts), 3), "cycles": rep["cycles"],
                          "coarse_iters": rep["coarse_iters"], "rel": [x / h[0] for x in h]}), flush=True)
        s.close()
