"""Pins for the oracle's element-centred block smoother (oracle/ecsmoother.py; SURVEY 8(f) NEXT-4,
P:390-417).  The routes to the block inverse are independent: the literal slice R_i H_hat R_i^T
of the assembled global condensed operator, the assembly from the 27 element Schur complements,
the Schur complement of the assembled UNcondensed tensor-product block (interiors eliminated),
and the six-face fast-diagonalisation algorithm the GPU kernel follows."""
import numpy as np
import pytest

from oracle import condensed, ecsmoother as ec, mesh, mg

import pmg_inputs as pi


def _mesh(p, k=(3, 4, 3), neumann=0):
    w = [np.linspace(0.8, 1.2, k[0]), np.full(k[1], 1.2 / k[1]), np.linspace(0.5, 1.0, k[2])]
    return mesh.Mesh(k, w, p, neumann=neumann)


BLOCKS = [(0, 0, 0), (1, 1, 1), (2, 3, 2), (1, 0, 2), (0, 2, 1), (2, 1, 0)]


@pytest.mark.parametrize("neu", [0, 0b101010, 0b111111])
@pytest.mark.parametrize("p", [2, 3, 4])
def test_block_routes_agree(p, neu):
    m = _mesh(p, neumann=neu)
    op = condensed.CondensedOperator(m, 0.7)
    Hs = op.assembled_condensed()
    r = np.random.default_rng(p + neu).standard_normal(m.ntot) * m.free_skel
    for e in BLOCKS:
        pts, loc = ec.ec_points(m, e)
        A = ec.ec_matrix_block(op, e, pts)
        B = Hs[pts][:, pts].toarray()
        C = ec.ec_matrix_schur(op, e, loc)
        sc = np.abs(A).max()
        assert np.abs(A - B).max() <= 1e-13 * sc
        assert np.abs(A - C).max() <= 1e-12 * sc
        assert np.abs(A - A.T).max() <= 1e-14 * sc                       # symmetric
        assert np.linalg.eigvalsh(A).min() > 0                           # positive definite
        x = np.linalg.solve(A, r[pts])
        _, xt = ec.tpc_ec_inverse(op, e, r)
        assert np.abs(xt - x).max() <= 1e-12 * np.abs(x).max()


def test_block_points_are_the_six_face_planes():
    """Interior element of a 5^3 mesh: 6 planes of n_S^2 points minus the 12 shared lines counted
    twice plus the 8 triple points (inclusion-exclusion), n_S = 3p - 1."""
    p = 3
    n = ec.ec_n(p)
    m = mesh.Mesh((5, 5, 5), [np.ones(5)] * 3, p)
    pts, loc = ec.ec_points(m, (2, 2, 2))
    assert len(pts) == 6 * n * n - 12 * n + 8
    assert len(set(pts.tolist())) == len(pts)
    cl, ch = ec.ec_planes(p)
    assert all(((np.array(j) == cl) | (np.array(j) == ch)).any() for j in zip(*loc))


def test_whole_mesh_block_is_the_exact_solve():
    """On a 3^3 Dirichlet mesh the centre element's block covers every condensed unknown (its six
    planes are the whole interior skeleton): the fast block inverse is the exact condensed solve."""
    m = mesh.Mesh((3, 3, 3), [[0.3, 0.5, 0.4], [0.6, 0.2, 0.5], [0.4, 0.4, 0.7]], 4)
    op = condensed.CondensedOperator(m, 1.3)
    pts, _ = ec.ec_points(m, (1, 1, 1))
    fs = np.nonzero(m.free_skel)[0]
    assert np.array_equal(np.sort(pts), fs)
    r = np.random.default_rng(4).standard_normal(m.ntot) * m.free_skel
    Hs = op.assembled_condensed()
    x = np.zeros(m.ntot)
    x[fs] = np.linalg.solve(Hs[fs][:, fs].toarray(), r[fs])
    p2, xt = ec.tpc_ec_inverse(op, (1, 1, 1), r)
    assert np.abs(xt - x[p2]).max() <= 1e-12 * np.abs(x).max()


@pytest.mark.parametrize("neu", [0, 0b000011, 0b111111])
def test_weights_partition_of_unity(neu):
    m = _mesh(4, k=(4, 3, 1), neumann=neu)
    tot = np.zeros(m.ntot)
    for e in ec.elements(m):
        pts, loc = ec.ec_points(m, e)
        if len(pts):
            np.add.at(tot, pts, ec.ec_weights(m, e, loc))
    fs = m.free_skel
    assert np.abs(tot[fs] - 1.0).max() < 1e-12
    assert np.all(tot[~fs] == 0)


def test_weights_shape():
    """omega_e: 1/2 on the centre element (interior node), 1/2 at its faces, 0 at the block ends."""
    m = _mesh(5, k=(5, 5, 5))
    e = (2, 2, 2)
    g = ec.ec_index_range(m, e, 0)
    w = ec.ec_weight_1d(m, e, 0, g)
    cl, ch = ec.ec_planes(m.p)
    assert abs(w[cl] - 0.5) < 1e-13 and abs(w[ch] - 0.5) < 1e-13 and abs(w[cl + 2] - 0.5) < 1e-13
    assert w[0] < 1e-2 and w[-1] < 1e-2 and np.all(w >= 0)       # w(t) ~ 35 (1-t)^4 near the ends


@pytest.mark.parametrize("k,p,lam,stretch", [((4, 4, 4), 4, 0.0, None), ((5, 3, 4), 3, 1.0, 1.5)])
def test_mg_with_element_centred_smoother_converges_faster_than_star(k, p, lam, stretch):
    """More overlap: per-cycle contraction at least as good as the star smoother's,
    and the 1e-10 reduction within the paper's handful of cycles."""
    case = pi.small_case(k, p, lam, stretch=stretch)
    out = {}
    for sm in ("star", "element"):
        H = mg.Hierarchy(case.k, case.widths, p, lam, smoother=sm, coarse_rtol=1e-10)
        m = H.levels[-1].mesh
        F = condensed.weak_rhs(m, np.random.default_rng(0).uniform(-1, 1, m.ntot))
        _, rep = H.solve(F, 1e-10)
        assert rep["converged"]
        out[sm] = rep
    assert out["element"]["cycles"] <= min(out["star"]["cycles"], 8), (out["element"]["cycles"], out["star"]["cycles"])
    assert out["element"]["rho"] <= out["star"]["rho"]
