"""Pins for periodic directions ("in the periodic case the ghost
elements stay part of the domain, requiring no change in the operator").  Direction bitmask: bit d
set = direction d is periodic; the last grid plane of a periodic direction duplicates plane 0."""
import math

import numpy as np
import pytest

from oracle import condensed, mesh, mg, smoother

import pmg_inputs as pi

MASKS = [0b001, 0b110, 0b111]


def _mesh(p, k, periodic, neumann=0):
    w = [np.linspace(0.8, 1.2, k[0]), np.full(k[1], 1.3 / k[1]), np.linspace(0.5, 1.0, k[2])]
    return mesh.Mesh(k, w, p, neumann=neumann, periodic=periodic)


def test_free_mask_and_wrapped_elements():
    m = _mesh(3, (2, 3, 2), 0b001)
    i1, i2, i3 = [a.ravel() for a in m.idx]
    want = (i1 < m.N[0] - 1) & (i2 > 0) & (i2 < m.N[1] - 1) & (i3 > 0) & (i3 < m.N[2] - 1)
    assert np.array_equal(m.free, want)
    # the last element in x reaches back to plane 0; no element touches the duplicate plane
    t1 = m.local_t[0]
    last = m.elem_idx[m.k[0] - 1]
    assert np.all(i1[last[t1 == m.p]] == 0)
    assert not np.any(i1[m.elem_idx.ravel()] == m.N[0] - 1)
    with pytest.raises(ValueError):
        mesh.Mesh((1, 2, 2), [[1.0], [0.5, 0.5], [0.5, 0.5]], 2, periodic=0b001)      # k_d >= 2
    with pytest.raises(ValueError):
        mesh.Mesh((2, 2, 2), [[0.5, 0.5]] * 3, 2, periodic=0b001, neumann=0b000001)   # not Neumann too


@pytest.mark.parametrize("per", MASKS)
@pytest.mark.parametrize("p", [2, 3, 4])
def test_star_routes_agree_periodic(p, per):
    """Stars that wrap around a periodic direction: block assembly = literal slice R H_hat R^T of the
    global periodic operator = Schur complement of the uncondensed block = Alg. 1 (TPC) = fast
    diagonalisation (TPF)."""
    m = _mesh(p, (3, 2, 2), per)
    lam = 0.7
    op = condensed.CondensedOperator(m, lam)
    Hs = op.assembled_condensed()
    r = np.random.default_rng(p + per).standard_normal(m.ntot) * m.free_skel
    for v in [(0, 0, 0), (2, 1, 1), (0, 1, 1), (2, 0, 1), (1, 1, 0), (1, 1, 1), (0, 1, 0)]:
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


@pytest.mark.parametrize("per", MASKS)
def test_partition_of_unity_periodic(per):
    m = _mesh(4, (3, 2, 2), per)
    tot = np.zeros(m.ntot)
    for v in smoother.vertices(m):
        pts, loc = smoother.star_points(m, v)
        if len(pts):
            np.add.at(tot, pts, smoother.star_weights(m, v, loc))
    fs = m.free_skel
    assert np.abs(tot[fs] - 1.0).max() < 1e-13
    assert np.all(tot[~fs] == 0)


@pytest.mark.parametrize("per,neu", [(0b001, 0), (0b111, 0), (0b011, 0b100000)])
def test_condense_solve_recover_equals_full_solve_periodic(per, neu):
    m = mesh.Mesh((2, 3, 2), [[0.4, 0.6], [0.5, 0.2, 0.3], [0.3, 0.9]], 3, neumann=neu, periodic=per)
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


def _manufactured_error(p, per):
    """lambda = 1, f = 4 u: all periodic on (0, 2 pi)^3 with u = cos x cos y cos z, or periodic x and
    Dirichlet y, z on (0, 2 pi) x (0, pi)^2 with u = cos x sin y sin z; max nodal error of the MG
    solve (duplicate planes included, filled from plane 0)."""
    k = (3, 2, 2)
    L = (2 * math.pi,) * 3 if per == 0b111 else (2 * math.pi, math.pi, math.pi)
    H = mg.Hierarchy(k, pi.uniform_widths(k, L), p, 1.0, periodic=per)
    m = H.levels[-1].mesh
    x1, x2, x3 = [m.coords[d][m.idx[d].ravel()] for d in range(3)]
    ue = np.cos(x1) * ((np.cos(x2) * np.cos(x3)) if per == 0b111 else (np.sin(x2) * np.sin(x3)))
    u, rep = H.solve(condensed.weak_rhs(m, 4.0 * ue), 1e-12)
    assert rep["converged"] and rep["cycles"] <= 8
    return np.abs(u - ue).max()


@pytest.mark.parametrize("per", [0b001, 0b111])
def test_manufactured_solution_spectral_decay_periodic(per):
    errs = [_manufactured_error(p, per) for p in (2, 4, 6, 8)]
    assert errs[-1] < 1e-5
    for a, b in zip(errs, errs[1:]):
        assert b < a / 8, errs


def test_translation_invariance_periodic():
    """Uniform elements, periodic in x: shifting the right-hand side by one element along x shifts the
    MG solution by one element (the operator, the star set and the V-cycle are shift-invariant)."""
    k = (4, 2, 3)
    H = mg.Hierarchy(k, pi.uniform_widths(k, (1.0, 0.7, 0.9)), 4, 0.3, periodic=0b001, coarse_rtol=1e-13)
    m = H.levels[-1].mesh
    p, N1 = m.p, m.N[0]
    f = np.random.default_rng(5).uniform(-1, 1, m.ntot)
    g = m.grid(f)[:, :, :N1 - 1]                      # the periodic unknown planes
    g2 = np.roll(g, p, axis=2)
    f2 = np.zeros_like(m.grid(f))
    f2[:, :, :N1 - 1] = g2
    f2[:, :, N1 - 1] = g2[:, :, 0]
    u1, r1 = H.solve(condensed.weak_rhs(m, m.fill_periodic(np.pad(g, ((0, 0), (0, 0), (0, 1))).ravel())), 1e-12)
    u2, r2 = H.solve(condensed.weak_rhs(m, f2.ravel()), 1e-12)
    a = np.roll(m.grid(u1)[:, :, :N1 - 1], p, axis=2)
    b = m.grid(u2)[:, :, :N1 - 1]
    assert r1["cycles"] == r2["cycles"]
    assert np.abs(a - b).max() <= 1e-10 * np.abs(a).max()


def test_mg_solve_periodic_converges_fast():
    k = (4, 4, 4)
    H = mg.Hierarchy(k, pi.uniform_widths(k, (1.0,) * 3), 4, 0.5, periodic=0b011)
    m = H.levels[-1].mesh
    F = condensed.weak_rhs(m, np.random.default_rng(0).uniform(-1, 1, m.ntot))
    _, rep = H.solve(F, 1e-10)
    assert rep["converged"] and rep["cycles"] <= 6, rep["cycles"]
