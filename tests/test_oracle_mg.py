"""Pins for the oracle's transfer operators, coarse CG and multigrid solver
(Alg. 3/4) against polynomial reproduction, the paper's printed iteration counts (Table
stretched_poly_iterations) and the spectral accuracy of the discretisation."""
import json
import math
import os

import numpy as np
import pytest

import pmg_inputs as pi
from oracle import condensed, mesh, mg, transfer

GOLD = os.path.join(os.path.dirname(__file__), "golden", "stretched_poly_iterations.json")


@pytest.mark.parametrize("pc,pf", [(2, 4), (4, 8), (2, 3), (4, 6)])
def test_prolongation_reproduces_polynomials(pc, pf):
    k = (2, 3, 2)
    w = [np.array([0.4, 0.6]), np.array([0.2, 0.5, 0.3]), np.array([0.7, 0.3])]
    mc, mf = mesh.Mesh(k, w, pc), mesh.Mesh(k, w, pf)
    T = transfer.Transfer(mc, mf)

    def poly(m):   # degree 2 per direction, zero on the box boundary
        x1, x2, x3 = m.coords
        g = lambda x, L: x * (L - x)
        return (g(x3, 1.0)[:, None, None] * g(x2, 1.0)[None, :, None] * g(x1, 1.0)[None, None, :]).ravel()

    uc = poly(mc) * mc.free_skel
    uf = poly(mf) * mf.free_skel
    assert np.abs(T.prolong(uc) - uf).max() < 1e-13
    rng = np.random.default_rng(0)
    a = rng.standard_normal(mc.ntot) * mc.free_skel
    b = rng.standard_normal(mf.ntot) * mf.free_skel
    assert abs(T.prolong(a) @ b - a @ T.restrict(b)) < 1e-12 * abs(a @ T.restrict(b))
    assert np.all(T.restrict(b)[~mc.free_skel] == 0)


def test_level_degrees():
    assert mg.level_degrees(2) == [2]
    assert mg.level_degrees(3) == [2, 3]
    assert mg.level_degrees(4) == [2, 4]
    assert mg.level_degrees(12) == [2, 4, 8, 12]
    assert mg.level_degrees(16) == [2, 4, 8, 16]
    assert mg.level_degrees(24) == [2, 4, 8, 16, 24]
    assert mg.level_degrees(32) == [2, 4, 8, 16, 32]


def test_pcg_solves_coarse_system():
    lv = mg.Level((3, 2, 3), [np.full(3, 1 / 3), np.full(2, 0.5), np.array([0.2, 0.3, 0.5])], 2, 0.0, 7)
    b = np.random.default_rng(2).standard_normal(lv.mesh.ntot) * lv.mesh.free_skel
    x, its = mg.pcg(lv, b, 1e-13, 1000)
    fs = np.nonzero(lv.mesh.free_skel)[0]
    Hs = lv.op.assembled_condensed()[fs][:, fs].toarray()
    assert np.abs(x[fs] - np.linalg.solve(Hs, b[fs])).max() < 1e-11 * np.abs(x).max()
    assert its <= len(fs)


def _iters(alpha, p):
    k = (8, 8, 8)
    w = [pi.geometric_widths(8, 2 * math.pi, alpha)] * 3
    H = mg.Hierarchy(k, w, p, 0.0)
    m = H.levels[-1].mesh
    f = np.random.default_rng(0).uniform(-1, 1, m.ntot)
    _, rep = H.solve(condensed.weak_rhs(m, f), 1e-10, max_cycles=60)
    return rep


@pytest.mark.parametrize("alpha,p", [(1, 4), (1, 8), (1.5, 4), (2, 4)])
def test_iteration_counts_match_paper_table(alpha, p):
    gold = json.load(open(GOLD))
    want = gold["MG"][str(alpha if alpha != 1 else 1)][gold["p"].index(p)]
    rep = _iters(alpha, p)
    assert rep["converged"]
    assert abs(rep["cycles"] - want) <= 1, (rep["cycles"], want)
    if alpha == 1:
        assert rep["rho"] < 1e-2          # rho of order 1e-4 for MG
        h = rep["history"]
        assert all(b < a for a, b in zip(h, h[1:]))


def test_single_level_solve_p2():
    """p = p0 = 2 (L = 0): the solve is the coarse CG on the residual equation (reading c-10b)."""
    k = (4, 4, 4)
    H = mg.Hierarchy(k, pi.uniform_widths(k, (1, 1, 1)), 2, 0.0)
    m = H.levels[0].mesh
    F = condensed.weak_rhs(m, np.random.default_rng(1).uniform(-1, 1, m.ntot))
    u, rep = H.solve(F, 1e-10)
    assert rep["converged"] and rep["cycles"] <= 3


def test_exact_solution_is_a_fixed_point():
    k = (3, 3, 3)
    H = mg.Hierarchy(k, pi.uniform_widths(k, (1, 1, 1)), 4, 1.0, coarse_rtol=1e-13)
    top = H.levels[-1]
    m = top.mesh
    fs = np.nonzero(m.free_skel)[0]
    f = np.random.default_rng(3).standard_normal(m.ntot) * m.free_skel
    Hs = top.op.assembled_condensed()[fs][:, fs].toarray()
    u = np.zeros(m.ntot)
    u[fs] = np.linalg.solve(Hs, f[fs])
    u2 = H.vcycle(u, f)
    assert np.abs(u2 - u).max() < 1e-11 * np.abs(u).max()


def test_spectral_convergence_manufactured():
    """Config 1 without noise: lambda = 1, f = 3 sin x sin y sin z on (0,2pi)^3 has the exact
    solution u = (3/4) sin x sin y sin z; the nodal max error must decay spectrally in p."""
    errs = []
    for p in (2, 4, 6, 8):
        case = pi.config(1)
        k = case.k
        H = mg.Hierarchy(k, case.widths, p, 1.0)
        m = H.levels[-1].mesh
        x1, x2, x3 = m.coords
        s = (np.sin(x3)[:, None, None] * np.sin(x2)[None, :, None] * np.sin(x1)[None, None, :]).ravel()
        u, rep = H.solve(condensed.weak_rhs(m, 3.0 * s), 1e-12)
        errs.append(np.abs(u - 0.75 * s).max())
    assert all(b < 0.2 * a for a, b in zip(errs, errs[1:])), errs
    assert errs[-1] < 1e-5


def _iters_krylov(alpha, p, schedule):
    k = (8, 8, 8)
    w = [pi.geometric_widths(8, 2 * math.pi, alpha)] * 3
    H = mg.Hierarchy(k, w, p, 0.0, schedule=schedule)
    m = H.levels[-1].mesh
    f = np.random.default_rng(0).uniform(-1, 1, m.ntot)
    _, rep = H.solve_ipcg(condensed.weak_rhs(m, f), 1e-10, max_iters=60)
    return rep


@pytest.mark.parametrize("solver,alpha,p", [("kMG", 1, 4), ("kMG", 1.5, 4), ("kMG", 2, 4), ("kvMG", 1, 4),
                                            ("kvMG", 1.5, 4)])
def test_krylov_iteration_counts_match_paper_table(solver, alpha, p):
    """Alg. 5 (ipCG with a V-cycle preconditioner) against the kMG / kvMG rows of
    Table tab:stretched_poly_iterations, +-1 as for MG."""
    gold = json.load(open(GOLD))
    want = gold[solver][str(alpha if alpha != 1 else 1)][gold["p"].index(p)]
    rep = _iters_krylov(alpha, p, 0 if solver == "kMG" else 1)
    assert rep["converged"]
    assert abs(rep["cycles"] - want) <= 1, (rep["cycles"], want)


def test_krylov_accelerates_on_stretched_mesh():
    """Krylov acceleration lowers the stretched-mesh iteration counts of MG."""
    H_mg = _iters(2, 4)
    H_k = _iters_krylov(2, 4, 0)
    assert H_k["cycles"] < H_mg["cycles"]


@pytest.mark.parametrize("schedule,ratio,limit", [(0, 1 / 8, 8 / 7), (1, 1 / 4, 4 / 3)])
def test_smoothing_schedule_effort_per_level(schedule, ratio, limit, monkeypatch):
    """P:557-558 (Sec. 4.4): with constant smoothing the effort of a coarser level is 1/8 of the next
    finer one (geometric series <= 8/7); with nu_pre,l = nu_post,l = 2^(L-l) it is 2 (1/2)^3 = 1/4
    (series <= 4/3), the finest level smoothing once before and once after.  Counted from
    the smoothing steps one oracle V-cycle actually performs (p = 16: L = 3, degrees 2, 4, 8, 16;
    the smoother costs O(p_l^3) per element).  A wrong exponent in the schedule (2^l,
    2^(L-l+1)) changes either the finest count or the ratio."""
    k = (2, 2, 2)
    H = mg.Hierarchy(k, pi.uniform_widths(k, (1.0, 1.0, 1.0)), 16, 0.0, schedule=schedule)
    calls = [0] * (H.L + 1)
    orig = H.smooth_step

    def counting(l, u, f):
        calls[l] += 1
        return orig(l, u, f)
    monkeypatch.setattr(H, "smooth_step", counting)
    f = np.random.default_rng(0).standard_normal(H.levels[-1].mesh.ntot) * H.levels[-1].mesh.free_skel
    H.vcycle(np.zeros_like(f), f)
    assert calls[H.L] == 2 and calls[0] == 0
    effort = [calls[l] * H.degrees[l] ** 3 for l in range(H.L + 1)]
    for l in range(2, H.L + 1):
        assert effort[l - 1] == ratio * effort[l], (calls, effort)
    assert sum(effort) / effort[H.L] < limit


@pytest.mark.parametrize("solver", ["kMG", "kvMG"])
def test_krylov_counts_p16_match_paper_table(solver):
    """Table tab:stretched_poly_iterations, alpha = 1, p = 16: kMG 3, kvMG 2 (+-1)."""
    gold = json.load(open(GOLD))
    want = gold[solver]["1"][gold["p"].index(16)]
    rep = _iters_krylov(1, 16, 0 if solver == "kMG" else 1)
    assert rep["converged"] and abs(rep["cycles"] - want) <= 1, (rep["cycles"], want)
