"""Probe: solve time split of the config-2 weak-scaling problems (16 x 16 x 16N, p = 8) on ONE GPU,
to estimate the replicated coarse solve's share at N GPUs (the fine work per GPU is that of N = 1)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1808_03595_b200 as pmg  # noqa: E402
import pmg_inputs as pi  # noqa: E402

for n in [1, 2, 4, 8]:
    k = (16, 16, 16 * n)
    w = [np.full(16, 1 / 16), np.full(16, 1 / 16), np.full(16 * n, 1 / 16)]
    c = pi.Case("weak%d" % n, k, w, 8, 0.0, "uniform", seed=1)
    s = pmg.Solver(k, w, 8, 0.0)
    L = s.nlevels - 1
    x = [s.grid_coords(L, d) for d in range(3)]
    F = s.new_grid()
    s.weak_rhs(torch.from_numpy(c.f_nodal(x)).cuda(), F)
    u = s.new_grid()
    for _ in range(2):
        s.solve(F, u, 1e-10)
    s.timing_enable(True)
    rep = s.solve(F, u, 1e-10)
    cg_ms, _ = s.timing_read(4)
    s.timing_enable(False)
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(s.stream)
    rep = s.solve(F, u, 1e-10)
    b.record(s.stream)
    b.synchronize()
    print(json.dumps({"n": n, "k": k, "solve_ms": a.elapsed_time(b), "coarse_ms": cg_ms, "cycles": rep["cycles"],
                      "coarse_iters": rep["coarse_iters"]}), flush=True)
    s.close()
