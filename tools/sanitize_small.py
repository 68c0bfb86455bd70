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
# round 2 kernels: p = 9..16 star / element / condensation (k_star16, k_elem16, k_cr16), p = 17..32
# (k_star_tm, k_elem_apply_t), p = 2 thread-per-star, periodic faces, the grid-layout h-multigrid at p = 2
run((2, 3, 2), 12, 0.0)
run((2, 2, 2), 9, 0.4)
run((2, 2, 2), 24, 0.0)
run((4, 4, 4), 2, 0.3)
run((4, 2, 4), 6, 0.0, periodic=0b101)
run((2, 2, 2), 12, 0.5, periodic=0b010)
run((8, 8, 8), 2, 0.0, coarse_solver=2)
os.environ["PMG_STAR_W_MIN"] = "0"
run((3, 3, 3), 4, 0.0)
