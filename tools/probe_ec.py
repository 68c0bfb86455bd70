"""Element-centred smoother (NEXT-4) vs vertex stars on BASELINE configs: cycles, per-cycle
contraction, solve time, and the finest-level sweep time (CUDA events around the colour launches)."""
import sys, os, json
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
import paper_1808_03595_b200 as pmg, pmg_inputs as pi

names = sys.argv[1:] or ["1", "2", "3:4", "3:16", "4"]
for nm in names:
    parts = nm.split(":")
    case = pi.config(int(parts[0]), p=int(parts[1])) if len(parts) > 1 else pi.config(int(parts[0]))
    for sm in (0, 1):
        s = pmg.Solver(case.k, case.widths, case.p, case.lam, smoother=sm)
        L = s.nlevels - 1
        x = [s.grid_coords(L, d) for d in range(3)]
        F = s.new_grid(); s.weak_rhs(torch.from_numpy(case.f_nodal(x)).cuda(), F)
        u = s.new_grid()
        for _ in range(2): s.solve(F, u, 1e-10)
        ts = []
        for _ in range(5):
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(s.stream); rep = s.solve(F, u, 1e-10); b.record(s.stream); b.synchronize(); ts.append(a.elapsed_time(b))
        s.timing_enable(True)
        s.solve(F, u, 1e-10)
        torch.cuda.synchronize()
        sw_ms, sw_n = s.timing_read(0)
        s.timing_enable(False)
        n_dof = case.k[0] * case.k[1] * case.k[2] * case.p ** 3
        print(json.dumps({"case": case.name, "smoother": ["star", "element"][sm], "solve_ms": round(sum(ts) / len(ts), 3),
                          "unknowns_per_s": n_dof / (sum(ts) / len(ts) * 1e-3), "cycles": rep["cycles"], "rho": rep["rho"],
                          "finest_sweep_ms": sw_ms / max(sw_n, 1), "sweeps": sw_n}), flush=True)
        s.close()
        del F, u
        torch.cuda.empty_cache()
