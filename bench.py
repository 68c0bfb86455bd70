"""Benchmark: unknowns/s of a 1e-10 residual-drop pMG solve (FP64) on B200, BASELINE.json metric.

One "step" = one full pmg_solve (Alg. 4: condense, V-cycles until ||r|| <= 1e-10 ||r_0||,
recover) of the workload, inputs resident in HBM.  Default workload: BASELINE configs[4], the
north star's scaling configuration -- Poisson, 64 x 64 x (8 N) elements, p = 16, f ~ U[-1,1] seed 4,
134 M unknowns per GPU (weak scaling, "cfg5_poisson_64x64x8N_p16"); --strong splits the whole
64^3-element problem (1.07e9 unknowns) over the N GPUs instead.  N > 1 runs the z-slab
decomposition (one process per GPU under torchrun, NCCL halo planes per operator, allreduced
norms, allgathered coarse right-hand side with a replicated coarse CG).
L2 (126 MB) is flushed between timed steps by writing a 512 MB buffer (outside the per-step
events); the vectors themselves (1.1 GB grid, 0.2 GB skeleton per vector) exceed L2 anyway.

  python bench.py [--gpus N --steps K --warmup W] [--config 5|4|3|2|1] [--p P] [--strong]
                  [--impl reference]

--impl reference times the CPU oracle (oracle/, test infrastructure) on the same workload: the
deliberately slow, plain program the GPU path is checked against.  For configs 4 and 5 (and any
workload over 2^22 unknowns) each step is one oracle solve of an 8 x 8 x 8-element sub-box with
the same degree, lambda and width sequence, reported per unknown ("oracle, extrapolated": the
sub-box's coarse solve is cheaper than the full problem's, which favours the oracle).  Under
torchrun (N > 1) only rank 0 runs it.
"""
import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import pmg_inputs as pi  # noqa: E402

FP64_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12   # 37.2: 64 FP64 FMA/clk/SM x 148 SMs x 1.965 GHz
METRIC = "unknowns/s for a 1e-10 residual-drop pMG solve (FP64); smoother % of HBM peak"


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


class ClockSampler:
    """SM clocks and throttle reasons polled through NVML every 2 ms during the timed region (the
    solve takes milliseconds, shorter than nvidia-smi's sampling period)."""

    def __init__(self, dev):
        self.dev = dev
        self.sm, self.mx, self.reasons = [], [], set()
        self.stop_ev = threading.Event()
        self.t = None

    def start(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.dev)
            names = {nv.nvmlClocksEventReasonHwSlowdown: "hw_slowdown",
                     nv.nvmlClocksEventReasonHwThermalSlowdown: "hw_thermal_slowdown",
                     nv.nvmlClocksEventReasonSwThermalSlowdown: "sw_thermal_slowdown",
                     nv.nvmlClocksEventReasonSwPowerCap: "sw_power_cap"}
            self.mx.append(float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)))

            def loop():
                while not self.stop_ev.is_set():
                    self.sm.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
                    r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                    for bit, name in names.items():
                        if r & bit:
                            self.reasons.add(name)
                    time.sleep(0.002)
            self.t = threading.Thread(target=loop, daemon=True)
            self.t.start()
        except Exception:
            self.t = None

    def stop(self):
        if self.t is None:
            return None
        self.stop_ev.set()
        self.t.join(timeout=5)
        if not self.sm:
            return None
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": max(self.mx), "reasons": sorted(self.reasons),
                "samples": len(self.sm), "source": "NVML, 2 ms period, during the timed steps"}


def dist_init():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def case_for(args, n_gpu):
    """The workload; for n_gpu > 1 the weak-scaling variant: n_gpu z-slabs of the one-GPU problem
    stacked along x3 (config 5: 64 x 64 x 8 n_gpu elements, BASELINE.json; other configs: k3 n_gpu),
    or with --strong (config 5 only) the whole 64^3-element problem split into n_gpu slabs."""
    if args.config == 5:
        if args.strong:
            k = (64, 64, 64)
            return pi.Case("cfg5_poisson_64x64x64_p16", k, pi.uniform_widths(k, (1.0, 1.0, 1.0)), 16, 0.0,
                           "uniform", seed=4)
        return pi.config(5, n_gpu=n_gpu)
    c = pi.config(args.config, p=args.p)
    if n_gpu > 1:
        k = (c.k[0], c.k[1], c.k[2] * n_gpu)
        w = [c.widths[0], c.widths[1], np.tile(c.widths[2], n_gpu)]
        c = pi.Case(c.name + "_weak%d" % n_gpu, k, w, c.p, c.lam, c.f_kind, seed=c.seed, amp=c.amp,
                    noise=c.noise, origin=c.origin)
    return c


SUBBOX = 8          # oracle baseline of large workloads: an 8 x 8 x 8-element sub-box
FULL_ORACLE_MAX = 1 << 22


def oracle_case(case):
    """The problem the oracle times for `case`: the case itself when small, else the sub-box of its
    first SUBBOX elements per direction (same p, lambda, widths, right-hand side recipe)."""
    if case.n_dof <= FULL_ORACLE_MAX:
        return case, "full"
    k = tuple(min(SUBBOX, kd) for kd in case.k)
    w = [np.asarray(case.widths[d][:k[d]]) for d in range(3)]
    sub = pi.Case(case.name + "_subbox%dx%dx%d" % k, k, w, case.p, case.lam, case.f_kind, seed=case.seed,
                  amp=case.amp, noise=case.noise, origin=case.origin)
    return sub, "sub"


def workload_config(case, ws, strong):
    """The config dict both arms print (identical keys and values)."""
    return {"workload": case.name, "n_dof": case.n_dof, "p": case.p, "k": list(case.k), "lambda": case.lam,
            "rtol": 1e-10, "n_ranks": ws, "decomposition": ("z-slabs" if ws > 1 else "none"),
            "scaling_mode": "strong" if strong else "weak",
            "l2": "flushed between steps (512 MB write, outside the timed events); grid vectors exceed L2"}


def n_stars(case):
    k = case.k
    return (k[0] + 1) * (k[1] + 1) * (k[2] + 1) - 8


def n_skel_free(case):
    p, k = case.p, case.k
    m = p - 1
    full = (k[0] * p - 1) * (k[1] * p - 1) * (k[2] * p - 1)
    return full - k[0] * k[1] * k[2] * m ** 3


def oracle_solve_timer(case, reps, warm=0, smoother="star"):
    """Time full oracle solves (setup excluded) on the host cores; returns (seconds per solve, cycles)."""
    from oracle import condensed, mg
    H = mg.Hierarchy(case.k, case.widths, case.p, case.lam, smoother=smoother)
    m = H.levels[-1].mesh
    F = condensed.weak_rhs(m, case.f_nodal(m.coords))
    for _ in range(warm):
        H.solve(F, 1e-10)
    ts, cyc = [], 0
    for _ in range(reps):
        t0 = time.perf_counter()
        _, rep = H.solve(F, 1e-10)
        ts.append(time.perf_counter() - t0)
        cyc = rep["cycles"]
    return ts, cyc


def oracle_baseline(case, reps, warm=0, smoother="star"):
    """cpu_baseline / reference-arm measurement: (unknowns/s, seconds per timed solve, cycles, kind, sample)."""
    oc, mode = oracle_case(case)
    ts, cyc = oracle_solve_timer(oc, reps, warm=warm, smoother=smoother)
    t = statistics.mean(ts)
    if mode == "full":
        return oc.n_dof / t, t, cyc, "oracle", "%d full oracle solves (dense Schur / dense-LU stars; setup excluded) of %s, %.2f s each, %d cycles" % (reps, oc.name, t, cyc)
    return (oc.n_dof / t, t, cyc, "oracle, extrapolated",
            "%d oracle solves (setup excluded) of the %dx%dx%d-element sub-box of %s (same p, lambda, widths, "
            "f recipe; %d unknowns, %.2f s each, %d cycles), reported per unknown; the full problem's larger "
            "coarse solve is not included" % (reps, oc.k[0], oc.k[1], oc.k[2], case.name, oc.n_dof, t, cyc))


def cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def run_reference(args, ws, rank):
    if rank != 0:
        return 0
    case = case_for(args, ws)
    val, t, cyc, kind, sample = oracle_baseline(case, args.steps, warm=args.warmup)
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "unknowns/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": case.n_dof / val * 1e3, "higher_is_better": True,
        "scaling": "strong" if args.strong else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(case, ws, args.strong),
        "cpu_baseline": {"value": val, "unit": "unknowns/s", "cores": cores(), "kind": kind, "sample": sample},
        "e2e": {"value": val, "unit": "unknowns/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "solve": {"cycles": cyc, "seconds_per_timed_solve": t},
    }
    print(json.dumps(line))
    return 0


def load_traffic(case_name):
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        d = json.load(open(path))
        return d.get(case_name, {})
    except Exception:
        return {}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--strong", action="store_true", help="config 5: the whole 64^3 problem over N GPUs")
    ap.add_argument("--p", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--smoother", default="star", choices=["star", "element"],
                    help="vertex stars (Alg. 2, the headline) or element-centred blocks (NEXT-4)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    ws, rank, local = dist_init()
    if args.impl == "reference":
        return run_reference(args, ws, rank)

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_1808_03595_b200 as pmg

    case = case_for(args, ws)
    nccl_id = None
    if ws > 1:   # z-slab decomposition: the library's own NCCL communicator (id broadcast here)
        buf = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            buf.copy_(torch.frombuffer(bytearray(pmg.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(buf, 0)
        nccl_id = bytes(buf.cpu().numpy().tobytes())
    ec = args.smoother == "element"
    s = pmg.Solver(case.k, case.widths, case.p, case.lam, rank=rank, nranks=ws, nccl_id=nccl_id, smoother=1 if ec else 0)
    L = s.nlevels - 1
    coords = [s.grid_coords(L, d) for d in range(3)]
    f = torch.from_numpy(case.f_nodal(coords, i3_offset=s.slab["z0"] * case.p)).cuda()
    F = s.new_grid()
    s.weak_rhs(f, F)
    u = s.new_grid()
    stream = s.stream
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")   # 512 MB > 126 MB L2
    for _ in range(args.warmup):
        rep = s.solve(F, u, 1e-10)
    torch.cuda.synchronize()

    sampler = ClockSampler(local)
    sampler.start()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    # headline: K full solves, per-solve CUDA events on the library's stream, L2 flushed between
    l0 = s.launch_count()
    durs = []
    reps = []
    for _ in range(args.steps):
        flush.fill_(1.0)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        reps.append(s.solve(F, u, 1e-10))
        e1.record(stream)
        e1.synchronize()
        durs.append(e0.elapsed_time(e1))
    torch.cuda.synchronize()
    launches = s.launch_count() - l0
    if ws > 1:
        dist.barrier()
    clocks = sampler.stop()
    # kernel split (separate pass, not part of the headline): per-kernel events on the same stream
    s.timing_enable(True)
    for _ in range(args.steps):
        flush.fill_(1.0)
        s.solve(F, u, 1e-10)
    torch.cuda.synchronize()
    sm_ms, sm_n = s.timing_read(0)
    rs_ms, rs_n = s.timing_read(1)
    all_sm_ms, _ = s.timing_read(2)
    all_rs_ms, _ = s.timing_read(3)
    cg_ms, _ = s.timing_read(4)
    s.timing_enable(False)
    ms = statistics.mean(durs)
    if ws > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = case.n_dof / (ms / 1e3)          # all ranks' unknowns (case is the whole weak-scaled problem)

    # e2e: through the C ABI with host buffers (pinned), H2D of F and D2H of u inside the timed region
    e2e = None
    if not args.no_e2e:
        Fh = F.cpu().pin_memory()
        uh = torch.empty_like(Fh).pin_memory()
        ed = []
        for i in range(args.steps + 1):
            flush.fill_(1.0)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            s.solve_host(Fh, uh, 1e-10)
            e1.record(stream)
            e1.synchronize()
            if i > 0:
                ed.append(e0.elapsed_time(e1))
        ems = statistics.mean(ed)
        if ws > 1:
            t = torch.tensor([ems], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        nb = F.numel() * 8
        e2e = {"value": case.n_dof / (ems / 1e3), "unit": "unknowns/s", "ms_per_step": ems,
               "h2d_bytes_per_step": nb, "d2h_bytes_per_step": nb}

    # roofline of the dominant kernel: the star smoother (finest level), FP64-pipe bound
    sweep_ms = sm_ms / max(sm_n, 1)
    if ec:   # element-centred blocks: 73 n_S^3 per block, n_S = 3p - 1, one block per element
        n = 3 * case.p - 1
        flops = 73.0 * n ** 3 * case.k[0] * case.k[1] * case.k[2] / ws
    else:
        n = 2 * case.p - 1
        flops = 37.0 * n ** 3 * n_stars(case) / ws       # Alg. 1 count x stars per sweep (per rank)
    achieved = flops / (sweep_ms / 1e3) / 1e12
    bytes_alg = 24.0 * n_skel_free(case) / ws        # read r, read+write u, per rank
    peaks = measured_peaks()
    hbm = peaks.get("hbm_gbs", 6541.5)
    tr = load_traffic(case.name)
    traffic = tr.get("k_star_bytes_per_sweep")
    roof = {"kernel": ("k_ec_block_mma (27 colour launches = 1 element-centred sweep, finest level)" if ec else
                       "k_star (8 colour launches = 1 smoother sweep, finest level)"), "bound": "alu",
            "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s", "frac": achieved / FP64_PEAK_TFLOPS,
            "traffic": None if ec else traffic, "algorithmic_flops_per_sweep": flops, "sweep_ms": sweep_ms,
            "peak_source": "derived: 64 FP64 FMA/clk/SM x 148 SMs x 1.965 GHz (no FP64 entry in MEASURED_PEAKS.json); "
                           "measured DFMA microbenchmark 34.1 TFLOP/s (profiles/r01_step0_fp64_peaks.jsonl)",
            "hbm_view": {"achieved_gbs": bytes_alg / (sweep_ms / 1e3) / 1e9, "peak_gbs": hbm,
                         "frac": bytes_alg / (sweep_ms / 1e3) / 1e9 / hbm, "peak_source": "MEASURED_PEAKS.json hbm_gbs"}}
    res_ms = rs_ms / max(rs_n, 1)
    m = case.p - 1
    res_flops = (73.0 * m ** 3 + 24.0 * case.p * (case.p + 1) ** 2) * case.k[0] * case.k[1] * case.k[2] / ws
    residual = {"kernel": "k_elem_apply + k_gather_resid (finest level)", "ms": res_ms,
                "achieved_tflops": res_flops / (res_ms / 1e3) / 1e12,
                "achieved_gbs_alg": bytes_alg / (res_ms / 1e3) / 1e9}
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        val, t, cyc, kind, sample = oracle_baseline(case, 3, smoother=args.smoother)
        cpu = {"value": val, "unit": "unknowns/s", "cores": cores(), "kind": kind, "sample": sample}
    r = reps[-1]
    cfg = workload_config(case, ws, args.strong)
    if ec:
        cfg["workload"] += "_element_centred"
    line = {
        "metric": METRIC, "value": value, "unit": "unknowns/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong" if args.strong else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": cfg,
        "parallelism": ("single GPU" if ws == 1 else
                        "z-slab x%d (NCCL halo planes per operator, allreduce of owned norms, allgather of the "
                        "coarse RHS + replicated coarse CG)" % ws),
        "solve": {"smoother": args.smoother, "cycles": r["cycles"], "rho": r["rho"], "coarse_iters": r["coarse_iters"],
                  "phase_ms": {"condense": r["t_condense"], "cycles": r["t_cycles"], "coarse_cg": r["t_coarse"],
                               "recover": r["t_recover"]}},
        "roofline": roof,
        "residual_kernel": residual,
        "time_split_ms_per_step": {"smoother_all_levels": all_sm_ms / args.steps, "residual_all_levels": all_rs_ms / args.steps,
                                   "coarse_cg": cg_ms / args.steps},
        # the coarse CG is the largest single kernel at config 2 but is latency bound (no roofline
        # applies): one grid barrier (1.2 us measured, profiles/r01_gridsync.txt) per iteration
        "coarse_cg": {"share_of_step": (cg_ms / args.steps) / ms, "iterations_per_solve": r["coarse_iters"],
                      "us_per_iteration": 1e3 * (cg_ms / args.steps) / max(1, r["coarse_iters"]),
                      "bound": "latency: one grid barrier + two overlapped L2 round trips per iteration"},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clocks,
    }
    if rank == 0:
        print(json.dumps(line))
    s.close()
    if ws > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
