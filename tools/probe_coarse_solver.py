import sys, os, json
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np, torch
import paper_1808_03595_b200 as pmg, pmg_inputs as pi
case = pi.config(2)
for cs in (1, 2):
    s = pmg.Solver(case.k, case.widths, case.p, case.lam, coarse_solver=cs)
    L = s.nlevels - 1
    x = [s.grid_coords(L, d) for d in range(3)]
    F = s.new_grid(); s.weak_rhs(torch.from_numpy(case.f_nodal(x)).cuda(), F)
    u = s.new_grid()
    for _ in range(3): s.solve(F, u, 1e-10)
    ts = []
    for _ in range(10):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(s.stream); rep = s.solve(F, u, 1e-10); b.record(s.stream); b.synchronize(); ts.append(a.elapsed_time(b))
    print(json.dumps({"coarse_solver": cs, "ms": sum(ts) / len(ts), "coarse_iters": rep["coarse_iters"], "cycles": rep["cycles"]}))
    s.close()
