"""Pins for the oracle's star smoother: several independent routes to the same star
inverse, closed-form 1-D star matrices, partition of unity and convergence without relaxation."""
import math

import numpy as np
import pytest

from oracle import condensed, mesh, smoother


def _mesh(p, k=(2, 2, 2)):
    w = [np.linspace(0.8, 1.2, k[0]), np.full(k[1], 1.3 / k[1]), np.linspace(0.5, 1.0, k[2])]
    return mesh.Mesh(k, w, p)


def test_star_1d_closed_form_p2():
    """p = 2, h = 2: M = diag(4/3, 2/3, 4/3), K = [[8/3,-4/3,0],[-4/3,7/3,-4/3],[0,-4/3,8/3]],
    generalised eigenvalues (11 - sqrt 73)/4, 2, (11 + sqrt 73)/4 (derived by hand)."""
    m = mesh.Mesh((2, 2, 2), [np.full(2, 2.0)] * 3, 2)
    M, K, valid = smoother.star_1d(m, (1, 1, 1), 0)
    assert np.allclose(np.diag(M), [4 / 3, 2 / 3, 4 / 3], atol=1e-15)
    assert np.allclose(K, [[8 / 3, -4 / 3, 0], [-4 / 3, 7 / 3, -4 / 3], [0, -4 / 3, 8 / 3]], atol=1e-14)
    S, L = smoother._padded_fdm(M, K, valid)
    assert np.allclose(np.sort(L), [(11 - math.sqrt(73)) / 4, 2.0, (11 + math.sqrt(73)) / 4], atol=1e-13)
    assert np.allclose(S.T @ M @ S, np.eye(3), atol=1e-13)
    assert np.allclose(S.T @ K @ S, np.diag(L), atol=1e-13)


@pytest.mark.parametrize("p", [2, 3, 4, 5])
@pytest.mark.parametrize("lam", [0.0, 3.7])
def test_star_routes_agree(p, lam):
    m = _mesh(p, (3, 2, 2))
    op = condensed.CondensedOperator(m, lam)
    Hs = op.assembled_condensed()
    rng = np.random.default_rng(p)
    r = rng.standard_normal(m.ntot) * m.free_skel
    for v in [(1, 1, 1), (2, 1, 1), (0, 1, 1), (3, 0, 1), (1, 2, 2), (0, 0, 1), (3, 2, 1)]:
        pts, loc = smoother.star_points(m, v)
        A = smoother.star_matrix_block(op, v, pts)
        B = smoother.star_matrix_global(Hs, pts)
        C = smoother.star_matrix_schur(op, v, loc)
        sc = np.abs(A).max()
        assert np.abs(A - B).max() <= 1e-13 * sc
        assert np.abs(A - C).max() <= 1e-12 * sc
        assert np.abs(A - A.T).max() <= 1e-13 * sc
        x = np.linalg.solve(A, r[pts])
        _, x_tpc = smoother.tpc_star_inverse(op, v, r)
        _, x_tpf = smoother.tpf_star_inverse(op, v, r)
        assert np.abs(x_tpc - x).max() <= 1e-12 * np.abs(x).max()
        assert np.abs(x_tpf - x).max() <= 1e-12 * np.abs(x).max()


def test_star_counts_and_centre_star_is_global_inverse():
    """On a 2x2x2 Dirichlet mesh the centre star covers every free condensed unknown, so its
    inverse is the global H_hat^-1; unique star points = 3 n_S^2 - 3 n_S + 1."""
    p = 3
    m = _mesh(p)
    op = condensed.CondensedOperator(m, 0.0)
    pts, loc = smoother.star_points(m, (1, 1, 1))
    n = 2 * p - 1
    assert len(pts) == 3 * n * n - 3 * n + 1
    fs = np.nonzero(m.free_skel)[0]
    assert np.array_equal(np.sort(pts), fs)
    rng = np.random.default_rng(1)
    r = rng.standard_normal(m.ntot) * m.free_skel
    Hs = op.assembled_condensed()[fs][:, fs].toarray()
    x_glob = np.linalg.solve(Hs, r[fs])
    _, x_tpc = smoother.tpc_star_inverse(op, (1, 1, 1), r)
    order = np.argsort(pts)
    assert np.abs(x_tpc[order] - x_glob).max() <= 1e-12 * np.abs(x_glob).max()


@pytest.mark.parametrize("p", [2, 4, 5])
def test_weights_partition_of_unity(p):
    m = _mesh(p, (3, 3, 2))
    tot = np.zeros(m.ntot)
    for v in smoother.vertices(m):
        pts, loc = smoother.star_points(m, v)
        if len(pts):
            np.add.at(tot, pts, smoother.star_weights(m, v, loc))
    fs = m.free_skel
    assert np.abs(tot[fs] - 1.0).max() < 1e-13
    assert np.all(tot[~fs] == 0)
    # interior-vertex stars alone do NOT give a partition of unity (reading c-6)
    tot2 = np.zeros(m.ntot)
    for v in smoother.vertices(m):
        if all(0 < v[d] < m.k[d] for d in range(3)):
            pts, loc = smoother.star_points(m, v)
            np.add.at(tot2, pts, smoother.star_weights(m, v, loc))
    assert np.abs(tot2[fs] - 1.0).max() > 0.5


def test_smoother_converges_without_relaxation():
    """weighted additive Schwarz needs no relaxation factor; u <- u + S(f - H u)
    must reduce the residual monotonically on a uniform Dirichlet box."""
    m = mesh.Mesh((3, 3, 3), [np.full(3, 1 / 3)] * 3, 4)
    op = condensed.CondensedOperator(m, 0.0)
    sm = smoother.StarSmoother(op)
    assert sm.n_stars == 4 ** 3 - 8
    f = np.random.default_rng(5).standard_normal(m.ntot) * m.free_skel
    u = np.zeros(m.ntot)
    norms = []
    for _ in range(6):
        r = op.residual(u, f)
        norms.append(np.linalg.norm(r))
        u = u + sm.apply(r)
    assert all(b < a for a, b in zip(norms, norms[1:]))
    assert norms[-1] < 0.05 * norms[0]
    # correction vanishes on Dirichlet points
    assert np.all(sm.apply(f)[~m.free_skel] == 0)
