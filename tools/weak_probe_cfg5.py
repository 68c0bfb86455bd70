"""Probe: the config-5 weak-scaling problems (64 x 64 x 8N elements, p = 16, BASELINE.json) solved
on ONE GPU for N = 1, 2, 4, 8, to project the z-slab weak scaling: at N GPUs each rank does the
fine-level work of N = 1 (its slab) plus the replicated coarse solve of the whole N problem (the
coarse right-hand side is allgathered and every rank runs the same coarse CG),
plus one halo plane exchange per operator.  Reported per N: whole-solve time on one GPU, the
coarse-solve time (pmg_report t_coarse), cycles, and the projected per-GPU time
  t_proj(N) = [t_solve(1) - t_coarse(1)] + t_coarse(N) + t_halo(N),
t_halo from the halo bytes per solve (two record planes per operator call at 64 x 64 x p = 16,
~23.6 MB each) over the NVLink 5 unidirectional 900 GB/s (a lower bound on the exchange time,
not overlapped), and the projected weak-scaling efficiency t_proj(1) / t_proj(N)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1808_03595_b200 as pmg  # noqa: E402
import pmg_inputs as pi  # noqa: E402

rows = []
for n in [1, 2, 4, 8]:
    case = pi.config(5, n_gpu=n)
    s = pmg.Solver(case.k, case.widths, case.p, case.lam)
    L = s.nlevels - 1
    x = [s.grid_coords(L, d) for d in range(3)]
    F = s.new_grid()
    f = s.new_grid()
    plane = len(x[0]) * len(x[1])
    for z0 in range(0, len(x[2]), 64):
        z1 = min(z0 + 64, len(x[2]))
        f[z0 * plane:z1 * plane] = torch.from_numpy(case.f_nodal([x[0], x[1], x[2][z0:z1]], i3_offset=z0)).cuda()
    s.weak_rhs(f, F)
    del f
    u = s.new_grid()
    for _ in range(2):
        s.solve(F, u, 1e-10)
    ts, tc = [], []
    for _ in range(3):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(s.stream)
        rep = s.solve(F, u, 1e-10)
        b.record(s.stream)
        b.synchronize()
        ts.append(a.elapsed_time(b))
        tc.append(rep["t_coarse"])
    # halo traffic per solve: exchanges of one record plane in each direction per operator call on the
    # finest level (residual: u before, r after; smoother: u after) -- per V-cycle 3 residuals + 2 sweeps
    RS = 3 * 15 * 15 + 3 * 15 + 1
    plane_bytes = 65 * 65 * RS * 8
    calls = 1 + rep["cycles"] * (3 * 2 + 2)
    halo_ms = (0 if n == 1 else 2 * calls * plane_bytes / 900e9 * 1e3)
    row = {"n": n, "k": list(case.k), "n_dof": case.n_dof, "solve_ms_one_gpu": min(ts), "coarse_ms": min(tc),
           "cycles": rep["cycles"], "coarse_iters": rep["coarse_iters"], "halo_ms_lower_bound": halo_ms}
    rows.append(row)
    s.close()
    torch.cuda.empty_cache()
fine1 = rows[0]["solve_ms_one_gpu"] - rows[0]["coarse_ms"]
for r in rows:
    r["projected_ms_per_gpu"] = fine1 + r["coarse_ms"] + r["halo_ms_lower_bound"]
    r["projected_weak_efficiency"] = (fine1 + rows[0]["coarse_ms"]) / r["projected_ms_per_gpu"]
    print(json.dumps(r), flush=True)
