import os, sys, traceback
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import pmg_inputs as pi
import paper_1808_03595_b200 as pmg
for cfgname, case in [("small", pi.small_case((3, 2, 3), 4, 1.7, stretch=1.6)), ("cfg2", pi.config(2))]:
    outs = {}
    for env in ("0", "1"):
        os.environ["PMG_COARSE_CLUSTER"] = env
        try:
            s = pmg.Solver(case.k, case.widths, case.p, case.lam, coarse_rtol=1e-13)
            L = s.nlevels - 1
            n = s.level_info(L)[1]
            g = torch.from_numpy(np.random.default_rng(0).standard_normal(s.level_info(L)[2])).cuda()
            f = s.new_skel(L); s.skel_from_grid(L, g, f)
            u = s.new_skel(L)
            s.vcycle(u, f)
            torch.cuda.synchronize()
            outs[env] = u.cpu().numpy()
            print(cfgname, "cluster", env, "norm", np.linalg.norm(outs[env]), flush=True)
            s.close()
        except Exception as e:
            traceback.print_exc()
    if len(outs) == 2:
        print(cfgname, "rel diff", np.linalg.norm(outs["0"] - outs["1"]) / np.linalg.norm(outs["0"]), flush=True)
