"""GPU iteration counts for Table tab:stretched_poly_iterations (MG / kMG / kvMG x
alpha in {1, 1.5, 2} x p in {4, 8, 16, 32}, 8^3 elements on (0, 2 pi)^3, lambda = 0, random RHS,
1e-10 drop) and the anisotropic sweep of Sec. 5.3 (8^3 elements, p = 16, domain
(0, 2 pi AR) x (0, pi ceil(AR / 2)) x (0, 2 pi)).  One JSON line per run.

    python tools/probe_tables.py [table|ar|both]
"""
import json
import math
import os
import sys
import time

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1808_03595_b200 as pmg  # noqa: E402
import pmg_inputs as pi  # noqa: E402

SOLVERS = {"MG": dict(solver=0, schedule=0), "kMG": dict(solver=1, schedule=0), "kvMG": dict(solver=1, schedule=1)}


def run(k, widths, p, solver, max_cycles=200):
    s = pmg.Solver(k, widths, p, 0.0, **SOLVERS[solver])
    f = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, s.level_info(s.nlevels - 1)[2])).cuda()
    F = s.new_grid()
    s.weak_rhs(f, F)
    u = s.new_grid()
    t0 = time.perf_counter()
    rep = s.solve(F, u, 1e-10, max_cycles=max_cycles)
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    s.close()
    return rep, t


def table():
    gold = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden",
                                       "stretched_poly_iterations.json")))
    for alpha in (1, 1.5, 2):
        w = [pi.geometric_widths(8, 2 * math.pi, alpha)] * 3
        for p in (4, 8, 16, 32):
            for solver in SOLVERS:
                rep, t = run((8, 8, 8), w, p, solver)
                want = gold[solver][str(alpha)][gold["p"].index(p)]
                print(json.dumps({"probe": "table", "alpha": alpha, "p": p, "solver": solver, "iters": rep["cycles"],
                                  "paper": want, "converged": rep["converged"], "rho": rep["rho"], "s": t}), flush=True)


def ar():
    for AR in (1, 2, 4, 8, 16, 32, 48):
        L = (2 * math.pi * AR, math.pi * math.ceil(AR / 2), 2 * math.pi)
        w = pi.uniform_widths((8, 8, 8), L)
        for solver in SOLVERS:
            rep, t = run((8, 8, 8), w, 16, solver)
            print(json.dumps({"probe": "ar", "AR": AR, "p": 16, "solver": solver, "iters": rep["cycles"],
                              "converged": rep["converged"], "rho": rep["rho"], "s": t}), flush=True)


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "both"
    if what in ("table", "both"):
        table()
    if what in ("ar", "both"):
        ar()
