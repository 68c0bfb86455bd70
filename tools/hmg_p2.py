"""One p = 2 solve of the degree-sweep mesh (128^3 elements): the whole solve is the h-multigrid
preconditioned coarse CG (k_pcg_hmg_p2).  Profiling driver."""
import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
import paper_1808_03595_b200 as pmg, pmg_inputs as pi
p = int(sys.argv[1]) if len(sys.argv) > 1 else 2
case = pi.config(3, p=p)
s = pmg.Solver(case.k, case.widths, case.p, case.lam)
L = s.nlevels - 1
x = [s.grid_coords(L, d) for d in range(3)]
F = s.new_grid(); s.weak_rhs(torch.from_numpy(case.f_nodal(x)).cuda(), F)
u = s.new_grid()
rep = s.solve(F, u, 1e-10)
torch.cuda.synchronize()
print("ok", rep["cycles"], rep.get("coarse_iters"))
