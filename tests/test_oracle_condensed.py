"""Pins for the oracle's element operator and static condensation by brute force."""
import numpy as np
import pytest
import scipy.sparse.linalg as spla

from oracle import condensed, mesh
from oracle.gll import gll


@pytest.mark.parametrize("h", [(1.0, 1.0, 1.0), (0.3, 1.7, 0.9)])
@pytest.mark.parametrize("lam", [0.0, 2.5])
def test_element_energy_of_coordinate_functions(h, lam):
    """u = x_d on [0,h1]x[0,h2]x[0,h3]: u^T H_e u = V (1 + lam h_d^2 / 3) (GLL exact for degree 2).
    A coefficient attached to the wrong direction (g_1 vs g_3 of Eq. helmholtzop) fails this."""
    p = 3
    H = condensed.element_operator(p, h, lam)
    xi, _ = gll(p)
    t = np.arange(p + 1)
    t3, t2, t1 = [a.ravel() for a in np.meshgrid(t, t, t, indexing="ij")]
    V = h[0] * h[1] * h[2]
    for d, td in enumerate((t1, t2, t3)):
        u = 0.5 * (xi[td] + 1) * h[d]
        assert u @ H @ u == pytest.approx(V * (1 + lam * h[d] ** 2 / 3), rel=1e-12)
    assert np.allclose(H, H.T, atol=1e-12)


@pytest.mark.parametrize("p", [2, 3, 5])
def test_condensed_element_properties(p):
    m = mesh.Mesh((1, 1, 1), [[0.7], [1.2], [0.5]], p)
    for lam in (0.0, 3.0):
        blk = condensed.ElementBlocks(p, (0.7, 1.2, 0.5), lam, m.loc_B, m.loc_I)
        assert np.allclose(blk.Hhat, blk.Hhat.T, atol=1e-12 * np.abs(blk.Hhat).max())
        ev = np.linalg.eigvalsh(blk.Hhat)
        if lam == 0.0:
            assert np.abs(blk.Hhat @ np.ones(len(m.loc_B))).max() < 1e-11 * np.abs(blk.Hhat).max()
            assert ev[0] > -1e-11 and ev[1] > 1e-8
        else:
            assert ev[0] > 0


@pytest.mark.parametrize("p,lam", [(2, 0.0), (3, 1.5), (4, 0.0)])
def test_condense_solve_recover_equals_full_solve(p, lam):
    """condense -> dense condensed solve -> recover == dense solve of the full system (2^3 mesh)."""
    m = mesh.Mesh((2, 2, 2), [[0.4, 0.6], [0.5, 0.5], [0.3, 0.9]], p)
    op = condensed.CondensedOperator(m, lam)
    rng = np.random.default_rng(3)
    F = rng.standard_normal(m.ntot) * m.free
    A = op.assembled_full()
    fr = np.nonzero(m.free)[0]
    u_full = np.zeros(m.ntot)
    u_full[fr] = np.linalg.solve(A[fr][:, fr].toarray(), F[fr])
    Hs = op.assembled_condensed()
    fs = np.nonzero(m.free_skel)[0]
    fhat = op.condense(F)
    uh = np.zeros(m.ntot)
    uh[fs] = np.linalg.solve(Hs[fs][:, fs].toarray(), fhat[fs])
    u = op.recover(uh, F)
    assert np.abs(u - u_full).max() <= 1e-11 * np.abs(u_full).max()
    # the matrix-free apply equals the assembled condensed matrix
    x = rng.standard_normal(m.ntot) * m.free_skel
    assert np.allclose(op.apply(x), (Hs @ x) * m.free_skel, atol=1e-12 * np.abs(Hs @ x).max())
    # global H_hat is symmetric
    S = Hs[fs][:, fs]
    assert abs(S - S.T).max() <= 1e-12 * abs(S).max()


def test_diag_matches_assembled():
    m = mesh.Mesh((2, 3, 2), [[0.4, 0.6], [0.2, 0.5, 0.3], [0.3, 0.9]], 2)
    op = condensed.CondensedOperator(m, 0.5)
    d = op.diag()
    Hs = op.assembled_condensed()
    assert np.allclose(d, Hs.diagonal() * m.free_skel, rtol=1e-13, atol=0)


def test_weak_rhs_separable_equals_element_loop():
    m = mesh.Mesh((2, 3, 2), [[0.4, 0.6], [0.2, 0.5, 0.3], [0.3, 0.9]], 3)
    f = np.random.default_rng(0).standard_normal(m.ntot)
    assert np.allclose(condensed.weak_rhs(m, f), condensed._weak_rhs_loop(m, f), rtol=1e-13, atol=1e-15)
    # total lumped mass = volume of the box (1.0 x 1.0 x 1.2)
    vol = np.prod([condensed.lumped_mass_1d(m, d).sum() for d in range(3)])
    assert vol == pytest.approx(1.0 * 1.0 * 1.2, rel=1e-14)
