"""Pins for the oracle's h-multigrid coarse preconditioner (oracle/hmg.py; SURVEY 8(f) NEXT-2,
P:559-561, reading R16)."""
import numpy as np
import pytest

import pmg_inputs as pi
from oracle import condensed, hmg, mg

STRETCH = [np.array([0.3, 0.5, 0.2, 0.4]), np.full(4, 0.25), np.array([0.1, 0.3, 0.3, 0.5])]


def _lin(mesh):
    X = [mesh.coords[d][mesh.idx[d].ravel()] for d in range(3)]
    return 0.3 + 1.1 * X[0] - 0.7 * X[1] + 0.4 * X[2]


def test_prolongation_reproduces_linears():
    """With lambda = 0 a linear function is discretely harmonic inside every coarse element, so the
    quadratic interpolation + harmonic extension of its coarse skeleton values is exact on the fine
    skeleton (all faces Neumann: no boundary value is dropped; stretched widths)."""
    k = (4, 4, 4)
    mf = hmg.HLevel(k, STRETCH, 0.0, 63).mesh
    mc = hmg.HLevel((2, 2, 2), hmg.merged_widths(STRETCH), 0.0, 63).mesh
    P = hmg.h_prolongation(mc, mf, 0.0)
    assert np.abs(P @ (_lin(mc) * mc.free_skel) - _lin(mf) * mf.free_skel).max() < 1e-13
    # but not a generic quadratic (the centre value is the harmonic extension, not the quadratic)
    X = mf.coords[0][mf.idx[0].ravel()]
    Xc = mc.coords[0][mc.idx[0].ravel()]
    assert np.abs(P @ (Xc ** 2 * mc.free_skel) - X ** 2 * mf.free_skel).max() > 1e-3


@pytest.mark.parametrize("neu,lam", [(0, 0.0), (0b110011, 0.8)])
def test_vcycle_is_symmetric_positive_definite(neu, lam):
    """CG needs a symmetric positive-definite preconditioner: <V a, b> = <a, V b>, <V a, a> > 0."""
    k = (8, 8, 4)
    H = hmg.HMultigrid(k, pi.uniform_widths(k, (1.0, 1.0, 0.5)), lam, neu)
    fs = H.levels[0].mesh.free_skel
    rng = np.random.default_rng(2)
    a = rng.standard_normal(fs.size) * fs
    b = rng.standard_normal(fs.size) * fs
    va, vb = H.vcycle(a), H.vcycle(b)
    assert abs(va @ b - a @ vb) <= 1e-12 * abs(va @ b)
    assert va @ a > 0 and vb @ b > 0


def test_hmg_pcg_solves_and_is_mesh_independent():
    """The preconditioned coarse CG reaches the tolerance with a solution equal to a dense solve, in
    a number of iterations independent of the element count -- unlike Jacobi-PCG."""
    its_h, its_j = [], []
    for n in (4, 8, 16):
        k = (n, n, n)
        w = pi.uniform_widths(k, (1.0,) * 3)
        H = hmg.HMultigrid(k, w, 0.0)
        lv = H.levels[0]
        b = np.random.default_rng(n).standard_normal(lv.mesh.ntot) * lv.mesh.free_skel
        x, it = hmg.pcg_hmg(lv, H, b, 1e-10, 200)
        its_h.append(it)
        if n == 4:
            fs = np.nonzero(lv.mesh.free_skel)[0]
            A = lv.op.assembled_condensed()[fs][:, fs].toarray()
            xd = np.linalg.solve(A, b[fs])
            assert np.abs(x[fs] - xd).max() <= 1e-8 * np.abs(xd).max()
        if n <= 8:
            its_j.append(mg.pcg(mg.Level(k, w, 2, 0.0, 7), b, 1e-10, 10000)[1])
    # at 4^3 the level itself is small enough for the exact coarsest solve (one iteration)
    assert its_h[0] <= 2 and max(its_h[1:]) <= 16 and abs(its_h[2] - its_h[1]) <= 3, its_h
    assert its_j[1] > 1.5 * its_j[0]                 # Jacobi-PCG grows with the element count


def test_solve_with_hmg_coarse_solver_matches_jacobi():
    """The outer MG iteration does not care which CG solves its coarse level to the tolerance."""
    k = (8, 8, 8)
    w = pi.uniform_widths(k, (1.0,) * 3)
    outs = []
    for cs in ("jacobi", "hmg"):
        H = mg.Hierarchy(k, w, 4, 0.0, coarse_solver=cs, coarse_rtol=1e-12)
        m = H.levels[-1].mesh
        F = condensed.weak_rhs(m, np.random.default_rng(0).uniform(-1, 1, m.ntot))
        outs.append(H.solve(F, 1e-10))
    (u1, r1), (u2, r2) = outs
    assert r1["cycles"] == r2["cycles"]
    assert np.linalg.norm(u1 - u2) <= 1e-9 * np.linalg.norm(u1)
