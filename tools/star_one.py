import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch, numpy as np
import paper_1808_03595_b200 as pmg, pmg_inputs as pi
case = pi.config(2)
s = pmg.Solver(case.k, case.widths, case.p, case.lam, smoother=0)
L = s.nlevels - 1
r = torch.randn(s.level_info(L)[1], dtype=torch.float64, device="cuda")
u = torch.zeros_like(r)
for _ in range(3): s.smooth(L, r, u)
torch.cuda.synchronize()
print("ok")
