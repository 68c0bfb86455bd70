"""Pins for homogeneous Neumann faces (boundary conditions enter
the star blocks only through which points are unknowns; Dirichlet points are decoupled by identity
padding, Neumann points stay in the star).  Face bitmask: bit 2d / 2d+1 = low / high face of
direction d is Neumann."""
import math

import numpy as np
import pytest

from oracle import condensed, mesh, mg, smoother

import pmg_inputs as pi

MASKS = [0b000001, 0b001100, 0b110000, 0b101010, 0b111111]


def _mesh(p, k, neumann):
    w = [np.linspace(0.8, 1.2, k[0]), np.full(k[1], 1.3 / k[1]), np.linspace(0.5, 1.0, k[2])]
    return mesh.Mesh(k, w, p, neumann=neumann)


def test_free_mask_counts():
    m = _mesh(3, (2, 2, 2), 0b111111)
    assert m.free.all()                                   # all-Neumann: every node is an unknown
    m = _mesh(3, (2, 2, 2), 0b000011)                     # Neumann at both x faces only
    i1, i2, i3 = [a.ravel() for a in m.idx]
    want = (i2 > 0) & (i2 < m.N[1] - 1) & (i3 > 0) & (i3 < m.N[2] - 1)
    assert np.array_equal(m.free, want)


@pytest.mark.parametrize("neu", MASKS)
@pytest.mark.parametrize("p", [2, 3, 4])
def test_star_routes_agree_with_neumann_faces(p, neu):
    """Boundary stars with Neumann faces: the block assembly, the literal slice of the global
    condensed operator, the Schur complement of the uncondensed block, Alg. 1 (TPC) and the fast
    diagonalisation (TPF) give the same star inverse."""
    m = _mesh(p, (3, 2, 2), neu)
    lam = 0.7
    op = condensed.CondensedOperator(m, lam)
    Hs = op.assembled_condensed()
    r = np.random.default_rng(p + neu).standard_normal(m.ntot) * m.free_skel
    for v in [(0, 0, 0), (3, 2, 2), (0, 1, 1), (3, 0, 1), (1, 2, 2), (1, 1, 1), (2, 0, 2)]:
        pts, loc = smoother.star_points(m, v)
        if len(pts) == 0:
            continue
        A = smoother.star_matrix_block(op, v, pts)
        B = smoother.star_matrix_global(Hs, pts)
        C = smoother.star_matrix_schur(op, v, loc)
        sc = np.abs(A).max()
        assert np.abs(A - B).max() <= 1e-13 * sc
        assert np.abs(A - C).max() <= 1e-12 * sc
        x = np.linalg.solve(A, r[pts])
        _, x_tpc = smoother.tpc_star_inverse(op, v, r)
        _, x_tpf = smoother.tpf_star_inverse(op, v, r)
        assert np.abs(x_tpc - x).max() <= 1e-12 * np.abs(x).max()
        assert np.abs(x_tpf - x).max() <= 1e-12 * np.abs(x).max()


@pytest.mark.parametrize("neu", MASKS)
def test_partition_of_unity_with_neumann_faces(neu):
    m = _mesh(4, (3, 3, 2), neu)
    tot = np.zeros(m.ntot)
    for v in smoother.vertices(m):
        pts, loc = smoother.star_points(m, v)
        if len(pts):
            np.add.at(tot, pts, smoother.star_weights(m, v, loc))
    fs = m.free_skel
    assert np.abs(tot[fs] - 1.0).max() < 1e-13
    assert np.all(tot[~fs] == 0)


@pytest.mark.parametrize("neu", [0b001100, 0b111111])
def test_condense_solve_recover_equals_full_solve_neumann(neu):
    m = mesh.Mesh((2, 2, 2), [[0.4, 0.6], [0.5, 0.5], [0.3, 0.9]], 3, neumann=neu)
    op = condensed.CondensedOperator(m, 1.3)
    rng = np.random.default_rng(3)
    F = rng.standard_normal(m.ntot) * m.free
    A = op.assembled_full()
    fr = np.nonzero(m.free)[0]
    u_full = np.zeros(m.ntot)
    u_full[fr] = np.linalg.solve(A[fr][:, fr].toarray(), F[fr])
    Hs = op.assembled_condensed()
    fs = np.nonzero(m.free_skel)[0]
    uh = np.zeros(m.ntot)
    uh[fs] = np.linalg.solve(Hs[fs][:, fs].toarray(), op.condense(F)[fs])
    u = op.recover(uh, F)
    assert np.abs(u - u_full).max() <= 1e-11 * np.abs(u_full).max()


def _manufactured_error(p, neu, kind):
    """lambda = 1 on (0, pi)^3: u = cos x cos y cos z (all Neumann) or u = sin x cos y cos z
    (Dirichlet at the x faces, Neumann elsewhere); f = 4 u; max nodal error of the MG solve."""
    k = (2, 2, 2)
    w = pi.uniform_widths(k, (math.pi,) * 3)
    H = mg.Hierarchy(k, w, p, 1.0, neumann=neu)
    m = H.levels[-1].mesh
    x1, x2, x3 = [m.coords[d][m.idx[d].ravel()] for d in range(3)]
    ue = (np.cos(x1) if kind == "cos" else np.sin(x1)) * np.cos(x2) * np.cos(x3)
    u, rep = H.solve(condensed.weak_rhs(m, 4.0 * ue), 1e-12)
    assert rep["converged"] and rep["cycles"] <= 8
    return np.abs(u - ue * m.free).max()


@pytest.mark.parametrize("neu,kind", [(0b111111, "cos"), (0b111100, "sin")])
def test_manufactured_solution_spectral_decay(neu, kind):
    errs = [_manufactured_error(p, neu, kind) for p in (2, 4, 6, 8)]
    assert errs[-1] < 1e-6
    for a, b in zip(errs, errs[1:]):
        assert b < a / 8, errs


def test_mg_solve_neumann_converges_fast():
    """Neumann faces change only which points are unknowns; the MG iteration keeps its few-cycle
    convergence on a uniform box."""
    k = (4, 4, 4)
    H = mg.Hierarchy(k, pi.uniform_widths(k, (1.0,) * 3), 4, 0.5, neumann=0b110011)
    m = H.levels[-1].mesh
    F = condensed.weak_rhs(m, np.random.default_rng(0).uniform(-1, 1, m.ntot))
    _, rep = H.solve(F, 1e-10)
    assert rep["converged"] and rep["cycles"] <= 6, rep["cycles"]
