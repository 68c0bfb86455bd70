"""Finest-level operators of the bench workload (config 5 slab: 64 x 64 x 8 elements, p = 16) for
ncu captures: a few smoother sweeps and residual evaluations on random skeleton vectors.

    python tools/cfg5_ops.py [--config 5] [--p P] [--reps 3]
"""
import argparse
import os
import sys

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_1808_03595_b200 as pmg  # noqa: E402
import pmg_inputs as pi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--p", type=int, default=None)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--solve", action="store_true", help="also one full solve (condense / recover kernels)")
a = ap.parse_args()
case = pi.config(a.config, p=a.p)
s = pmg.Solver(case.k, case.widths, case.p, case.lam)
L = s.nlevels - 1
n = s.level_info(L)[1]
r = torch.randn(n, dtype=torch.float64, device="cuda")
u = torch.zeros_like(r)
f = torch.randn_like(r)
q = torch.zeros_like(r)
for _ in range(a.reps):
    s.smooth(L, r, u)
    s.residual(L, u, f, q)
if a.solve:
    F = s.new_grid()
    F.copy_(torch.randn_like(F))
    ug = s.new_grid()
    s.solve(F, ug, 1e-10)
torch.cuda.synchronize()
print("ok", case.name, n)
