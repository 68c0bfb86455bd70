import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
import paper_1808_03595_b200 as pmg, pmg_inputs as pi
case = pi.config(2)
s = pmg.Solver(case.k, case.widths, case.p, case.lam)
L = s.nlevels - 1
u = torch.randn(s.level_info(L)[1], dtype=torch.float64, device="cuda")
f = torch.randn_like(u)
r = torch.zeros_like(u)
for _ in range(20): s.residual(L, u, f, r)
torch.cuda.synchronize()
print("ok")
