"""Degree sweep (BASELINE config 3): p = 2..32 at ~16.7 M unknowns (k = round(256/p)^3), lambda = 0,
f ~ N(0,1) seed 2.  Times the smoother sweep, the residual and the full solve separately (CUDA
events on the library's stream, after warm-up), one JSON line per degree.

    python tools/sweep.py [--p 2,4,8,...] [--steps 5] [--solve]
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1808_03595_b200 as pmg  # noqa: E402
import pmg_inputs as pi  # noqa: E402

FP64_PEAK = 148 * 64 * 2 * 1.965e9 / 1e12
HBM = 6530.0


def timed(stream, fn, reps):
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--p", default="2,4,8,12,16,24,32")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--solve", action="store_true")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    for p in [int(v) for v in args.p.split(",")]:
        case = pi.config(3, p=p)
        s = pmg.Solver(case.k, case.widths, case.p, case.lam)
        L = s.nlevels - 1
        st = s.stream
        u = s.new_skel(L)
        f = s.new_skel(L)
        r = s.new_skel(L)
        g = s.new_grid(L)
        g.copy_(torch.randn(g.numel(), dtype=torch.float64, generator=torch.Generator().manual_seed(p)))
        s.skel_from_grid(L, g, f)
        s.skel_from_grid(L, g, u)
        for _ in range(2):
            s.smooth(L, f, u)
            s.residual(L, u, f, r)
        torch.cuda.synchronize()
        t_sm = timed(st, lambda: s.smooth(L, f, u), args.steps)
        t_rs = timed(st, lambda: s.residual(L, u, f, r), args.steps)
        k = case.k
        n = 2 * p - 1
        m = p - 1
        nstars = (k[0] + 1) * (k[1] + 1) * (k[2] + 1) - 8
        nskel = (k[0] * p - 1) * (k[1] * p - 1) * (k[2] * p - 1) - k[0] * k[1] * k[2] * m ** 3
        fl_sm = 37.0 * n ** 3 * nstars
        fl_rs = (73.0 * m ** 3 + 24.0 * p * (p + 1) ** 2) * k[0] * k[1] * k[2]
        line = {"config": case.name, "p": p, "k": list(k), "n_dof": case.n_dof, "n_skel": nskel,
                "smoother_ms": t_sm, "smoother_tflops": fl_sm / t_sm / 1e9,
                "smoother_fp64_frac": fl_sm / t_sm / 1e9 / FP64_PEAK,
                "smoother_hbm_frac_alg": 24.0 * nskel / t_sm / 1e6 / HBM,
                "residual_ms": t_rs, "residual_tflops": fl_rs / t_rs / 1e9,
                "residual_fp64_frac": fl_rs / t_rs / 1e9 / FP64_PEAK,
                "residual_hbm_frac_alg": 24.0 * nskel / t_rs / 1e6 / HBM}
        if args.solve:
            coords = [s.grid_coords(L, d) for d in range(3)]
            fn = torch.from_numpy(case.f_nodal(coords)).cuda()
            F = s.new_grid()
            s.weak_rhs(fn, F)
            U = s.new_grid()
            rep = s.solve(F, U, 1e-10)
            t_solve = timed(st, lambda: s.solve(F, U, 1e-10), max(2, args.steps // 2))
            rep = s.solve(F, U, 1e-10)
            line.update({"solve_ms": t_solve, "cycles": rep["cycles"], "rho": rep["rho"],
                         "coarse_iters": rep["coarse_iters"], "unknowns_per_s": case.n_dof / t_solve * 1e3,
                         "ns_per_unknown": t_solve * 1e6 / case.n_dof})
        print(json.dumps(line), flush=True)
        s.close()
        del u, f, r, g
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
