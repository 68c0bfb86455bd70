"""Coarse solver probe: Jacobi-PCG vs h-multigrid-PCG coarse solves (solve time, coarse iterations,
cycles) per BASELINE config at the default coarse tolerance (reading R11 / R16)."""
import sys, os, json
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
import paper_1808_03595_b200 as pmg, pmg_inputs as pi

names = sys.argv[1:] or ["2", "3:4", "3:8", "3:16", "4", "5"]
for nm in names:
    parts = nm.split(":")
    case = pi.config(int(parts[0]), p=int(parts[1])) if len(parts) > 1 else pi.config(int(parts[0]))
    for cs in (1, 2):
        s = pmg.Solver(case.k, case.widths, case.p, case.lam, coarse_solver=cs)
        L = s.nlevels - 1
        x = [s.grid_coords(L, d) for d in range(3)]
        F = s.new_grid(); s.weak_rhs(torch.from_numpy(case.f_nodal(x)).cuda(), F)
        u = s.new_grid()
        for _ in range(2): s.solve(F, u, 1e-10)
        ts = []
        for _ in range(5):
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(s.stream); rep = s.solve(F, u, 1e-10); b.record(s.stream); b.synchronize(); ts.append(a.elapsed_time(b))
        print(json.dumps({"case": case.name, "coarse_solver": cs, "ms": round(sum(ts) / len(ts), 3),
                          "coarse_iters": rep["coarse_iters"], "cycles": rep["cycles"]}), flush=True)
        s.close()
        del F, u
        torch.cuda.empty_cache()
