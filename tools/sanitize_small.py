"""Tiny solves for compute-sanitizer (memcheck / racecheck): star and element-centred smoothers,
Krylov, Neumann, h-multigrid coarse solver, several degrees."""
import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np, torch
import paper_1808_03595_b200 as pmg, pmg_inputs as pi

def run(k, p, lam, **kw):
    case = pi.small_case(k, p, lam, stretch=1.3)
    s = pmg.Solver(case.k, case.widths, p, lam, **kw)
    L = s.nlevels - 1
    f = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, s.level_info(L)[2])).cuda()
    F = s.new_grid(); s.weak_rhs(f, F)
    u = s.new_grid()
    rep = s.solve(F, u, 1e-8, max_cycles=3)
    torch.cuda.synchronize()
    s.close()
    print(k, p, kw, rep["cycles"], flush=True)

run((3, 2, 3), 4, 0.5)
run((3, 3, 2), 8, 0.0)
run((2, 2, 2), 16, 1.0)
run((3, 2, 2), 5, 0.7, smoother=1)
run((2, 2, 2), 13, 0.7, smoother=1)
run((2, 2, 1), 16, 0.7, smoother=1)
run((3, 3, 3), 4, 0.2, solver=1, neumann=0b100101)
run((8, 8, 4), 4, 0.0, coarse_solver=2)
