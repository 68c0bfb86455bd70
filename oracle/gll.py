"""1-D ingredients (oracle; test infrastructure only).

P:85-86 (Sec. 2.1): "M_S is the one-dimensional standard element mass matrix, approximated
with GLL quadrature and K_S the standard element stiffness matrix", both (p+1)x(p+1).
P:439 (Sec. 4.1): the prolongation is "the embedded interpolation", built from 1-D
interpolation matrices.
P:312-316 (Sec. 3.2, Fig. weights): weight polynomials of degree p_W = 7, "one on the vertex
of the star and zero on all other vertices", "higher derivatives are zero at the vertices".
"""
import numpy as np


def legendre(p, x):
    """Legendre polynomial P_p(x) and P_{p-1}(x) by the three-term recurrence."""
    x = np.asarray(x, dtype=np.float64)
    p0 = np.ones_like(x)
    if p == 0:
        return p0, np.zeros_like(x)
    p1 = x.copy()
    for n in range(1, p):
        p0, p1 = p1, ((2 * n + 1) * x * p1 - n * p0) / (n + 1)
    return p1, p0


def gll(p):
    """GLL nodes (ascending, on [-1,1]) and weights for degree p >= 1.

    Nodes are -1, +1 and the roots of P_p'(x) (the zeros of (1-x^2) P_p'(x)); weights are
    w_i = 2 / (p (p+1) P_p(x_i)^2).  Newton iteration on x P_p - P_{p-1} = 0 (which vanishes at
    the same points) from the Chebyshev-Gauss-Lobatto guesses.
    """
    if p < 1:
        raise ValueError("GLL basis needs p >= 1")
    x = -np.cos(np.pi * np.arange(p + 1) / p)
    for _ in range(100):
        P, Pm1 = legendre(p, x)
        # f(x) = x P_p - P_{p-1} = (1-x^2) P_p' / p ; f'(x) = (p+1) P_p
        dx = (x * P - Pm1) / ((p + 1) * P)
        x = x - dx
        if np.max(np.abs(dx)) < 1e-16:
            break
    x[0], x[-1] = -1.0, 1.0
    x = 0.5 * (x - x[::-1])          # exact symmetry about 0
    P, _ = legendre(p, x)
    w = 2.0 / (p * (p + 1) * P ** 2)
    return x, w


def lagrange_eval(nodes, xs):
    """L[i, j] = l_j(xs[i]) for the Lagrange basis on ``nodes`` (plain product formula)."""
    nodes = np.asarray(nodes, dtype=np.float64)
    xs = np.asarray(xs, dtype=np.float64)
    n = len(nodes)
    L = np.ones((len(xs), n))
    for j in range(n):
        for k in range(n):
            if k != j:
                L[:, j] *= (xs - nodes[k]) / (nodes[j] - nodes[k])
    return L


def lagrange_deriv_at_nodes(nodes):
    """D[i, j] = l_j'(x_i): derivative of the product formula, evaluated term by term."""
    nodes = np.asarray(nodes, dtype=np.float64)
    n = len(nodes)
    D = np.zeros((n, n))
    for j in range(n):
        denom = np.prod([nodes[j] - nodes[k] for k in range(n) if k != j])
        for i in range(n):
            s = 0.0
            for m in range(n):
                if m == j:
                    continue
                prod = 1.0
                for k in range(n):
                    if k != j and k != m:
                        prod *= nodes[i] - nodes[k]
                s += prod
            D[i, j] = s / denom
    return D


def reference_matrices(p):
    """(nodes, weights, M_hat, K_hat) on [-1,1]: M_hat = diag(w) (GLL-lumped),
    K_hat[i,j] = sum_q w_q l_i'(x_q) l_j'(x_q)."""
    x, w = gll(p)
    D = lagrange_deriv_at_nodes(x)
    K = D.T @ np.diag(w) @ D
    K = 0.5 * (K + K.T)
    return x, w, np.diag(w), K


def element_matrices_1d(p, h):
    """Physical 1-D matrices of an element of width h: M = (h/2) M_hat, K = (2/h) K_hat.

    Equivalent to the coefficient vector g_e = (h1 h2 h3 / 8)(lambda, 4/h1^2, 4/h2^2, 4/h3^2)
    of Eq. (helmholtzop), distributed over the three Kronecker factors."""
    _, _, Mh, Kh = reference_matrices(p)
    return 0.5 * h * Mh, (2.0 / h) * Kh


def interpolation_matrix(p_coarse, p_fine):
    """J[i, a] = l_a^{(p_coarse)}(xi_i^{(p_fine)}): 1-D factor of the embedded interpolation
    (P:439)."""
    xc, _ = gll(p_coarse)
    xf, _ = gll(p_fine)
    return lagrange_eval(xc, xf)


def weight_poly_coeffs(pw=7):
    """Coefficients c[0..pw] (increasing powers) of the 1-D weight polynomial w(t), t in [0,1]
    the distance from the star's vertex in element units.

    P:313-315: one on the vertex (w(0) = 1), zero on the other vertex (w(1) = 0), and the
    higher derivatives zero at the vertices: w^(k)(0) = w^(k)(1) = 0 for k = 1..(pw-1)/2.
    For pw = 7 these are 8 conditions for 8 coefficients ("p_W = 7 was utilized").
    Solved here as a plain linear system (no closed form is assumed)."""
    if pw % 2 == 0:
        raise ValueError("weight degree must be odd")
    nd = (pw + 1) // 2
    A = np.zeros((pw + 1, pw + 1))
    b = np.zeros(pw + 1)
    row = 0
    for t0, val in ((0.0, 1.0), (1.0, 0.0)):
        for k in range(nd):
            for j in range(pw + 1):
                if j >= k:
                    coef = np.prod(np.arange(j - k + 1, j + 1, dtype=np.float64))
                    A[row, j] = coef * (t0 ** (j - k) if j - k > 0 else 1.0)
            b[row] = val if k == 0 else 0.0
            row += 1
    return np.linalg.solve(A, b)


def weight_poly(t, pw=7):
    c = weight_poly_coeffs(pw)
    t = np.asarray(t, dtype=np.float64)
    return sum(c[j] * t ** j for j in range(len(c)))
