"""Pins for the oracle's 1-D ingredients against closed forms."""
import math

import numpy as np
import pytest

from oracle import gll


def test_gll_p1_closed_form():
    x, w, M, K = gll.reference_matrices(1)
    assert np.allclose(x, [-1, 1], atol=0) and np.allclose(w, [1, 1], atol=1e-15)
    assert np.allclose(K, [[0.5, -0.5], [-0.5, 0.5]], atol=1e-15)


def test_gll_p2_closed_form():
    # GLL p=2: nodes {-1,0,1}, weights (1/3, 4/3, 1/3); K = (1/6)[[7,-8,1],[-8,16,-8],[1,-8,7]]
    x, w, M, K = gll.reference_matrices(2)
    assert np.allclose(x, [-1, 0, 1], atol=1e-16)
    assert np.allclose(w, [1 / 3, 4 / 3, 1 / 3], atol=1e-15)
    assert np.allclose(K, np.array([[7, -8, 1], [-8, 16, -8], [1, -8, 7]]) / 6, atol=1e-14)


def test_gll_p3_closed_form():
    # GLL p=3: interior nodes +-1/sqrt(5), weights (1/6, 5/6, 5/6, 1/6)
    x, w = gll.gll(3)
    assert np.allclose(x, [-1, -1 / math.sqrt(5), 1 / math.sqrt(5), 1], atol=1e-15)
    assert np.allclose(w, [1 / 6, 5 / 6, 5 / 6, 1 / 6], atol=1e-15)


@pytest.mark.parametrize("p", [1, 2, 3, 4, 7, 8, 16, 32])
def test_gll_quadrature_exact(p):
    x, w = gll.gll(p)
    assert abs(w.sum() - 2.0) < 1e-13
    assert np.all(np.diff(x) > 0)
    for k in range(2 * p):      # exact to degree 2p-1
        exact = 0.0 if k % 2 else 2.0 / (k + 1)
        assert abs(np.dot(w, x ** k) - exact) < 1e-13


@pytest.mark.parametrize("p", [2, 5, 8, 16])
def test_stiffness_properties(p):
    x, w, M, K = gll.reference_matrices(p)
    assert np.allclose(K, K.T, atol=1e-12)
    assert np.max(np.abs(K.sum(axis=1))) < 1e-11
    ev = np.linalg.eigvalsh(K)
    assert abs(ev[0]) < 1e-10 and ev[1] > 1e-6
    # K_ij = int l_i' l_j' exactly for polynomials: u = x^2 gives u^T K u = int (2x)^2 = 8/3
    u = x ** 2
    assert abs(u @ K @ u - 8.0 / 3.0) < 1e-11


@pytest.mark.parametrize("p", [2, 3, 8])
def test_derivative_matrix_exact_on_polynomials(p):
    x, _ = gll.gll(p)
    D = gll.lagrange_deriv_at_nodes(x)
    for k in range(p + 1):
        assert np.allclose(D @ x ** k, k * x ** max(k - 1, 0) if k else 0 * x, atol=1e-10)


def test_weight_polynomial_closed_form():
    # 8 Hermite conditions give 1 - 35 t^4 + 84 t^5 - 70 t^6 + 20 t^7
    c = gll.weight_poly_coeffs(7)
    assert np.allclose(c, [1, 0, 0, 0, -35, 84, -70, 20], atol=1e-10)
    t = np.linspace(0, 1, 101)
    assert np.allclose(gll.weight_poly(t) + gll.weight_poly(1 - t), 1.0, atol=1e-13)
    assert gll.weight_poly(0.0) == pytest.approx(1.0) and abs(gll.weight_poly(1.0)) < 1e-13


@pytest.mark.parametrize("pc,pf", [(2, 4), (4, 8), (8, 16), (2, 3), (4, 5)])
def test_interpolation_matrix(pc, pf):
    J = gll.interpolation_matrix(pc, pf)
    xc, _ = gll.gll(pc)
    xf, _ = gll.gll(pf)
    assert np.allclose(J.sum(axis=1), 1.0, atol=1e-13)
    assert np.array_equal(J[0], np.eye(pc + 1)[0]) and np.array_equal(J[-1], np.eye(pc + 1)[-1])
    for k in range(pc + 1):
        assert np.allclose(J @ xc ** k, xf ** k, atol=1e-12)
