"""Element Helmholtz operator, static condensation, condensed operator (oracle).

P:75-91 Eq. (helmholtzop): H_e = g0 M(x)M(x)M + g1 M(x)M(x)K + g2 M(x)K(x)M + g3 K(x)M(x)M,
  g_e = (h1 h2 h3 / 8)(lambda, 4/h1^2, 4/h2^2, 4/h3^2); the last Kronecker factor acts on x1.
P:93-122 (Sec. 2.2): H_hat = H_BB - H_BI H_II^-1 H_IB, F_hat = F_B - H_BI H_II^-1 F_I,
  u_I = H_II^-1 F_I - H_II^-1 H_IB u_B, and H_hat = sum_e Q_hat_e H_hat_e Q_hat_e^T.
P:132-134: r_hat = F_hat - H_hat u_hat.

Dense matrices only: H_e is built with np.kron and condensed by a dense Cholesky solve.
"""
import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp

from .gll import element_matrices_1d


def element_operator(p, h, lam):
    """Dense H_e (size (p+1)^3) for widths h = (h1, h2, h3), local order x1 fastest."""
    M1, K1 = element_matrices_1d(p, h[0])
    M2, K2 = element_matrices_1d(p, h[1])
    M3, K3 = element_matrices_1d(p, h[2])
    return (lam * np.kron(M3, np.kron(M2, M1)) + np.kron(M3, np.kron(M2, K1))
            + np.kron(M3, np.kron(K2, M1)) + np.kron(K3, np.kron(M2, M1)))


class ElementBlocks:
    """H_e split into boundary (B) / interior (I) blocks and its Schur complement H_hat_e."""

    def __init__(self, p, h, lam, loc_B, loc_I):
        H = element_operator(p, h, lam)
        self.HBB = H[np.ix_(loc_B, loc_B)]
        self.HBI = H[np.ix_(loc_B, loc_I)]
        self.HIB = H[np.ix_(loc_I, loc_B)]
        self.HII = H[np.ix_(loc_I, loc_I)]
        if len(loc_I):
            self.cho = sla.cho_factor(self.HII)
            self.Hhat = self.HBB - self.HBI @ sla.cho_solve(self.cho, self.HIB)
        else:
            self.cho = None
            self.Hhat = self.HBB.copy()
        self.Hhat = 0.5 * (self.Hhat + self.Hhat.T)
        self.H = H

    def solve_II(self, rhs):
        return sla.cho_solve(self.cho, rhs) if self.cho is not None else rhs


class CondensedOperator:
    """Global condensed operator on a Mesh, applied element by element."""

    def __init__(self, mesh, lam):
        if lam < 0:
            raise ValueError("lambda >= 0 required")
        self.mesh = mesh
        self.lam = float(lam)
        self.groups = []
        for h, elems in mesh.element_groups():
            blk = ElementBlocks(mesh.p, h, self.lam, mesh.loc_B, mesh.loc_I)
            self.groups.append((blk, elems))
        self._fs = mesh.free_skel.astype(np.float64)
        self._free = mesh.free.astype(np.float64)

    # --- condensed system -------------------------------------------------------------
    def apply(self, u):
        """H_hat u on free skeleton points (zero elsewhere)."""
        m = self.mesh
        u = np.asarray(u, dtype=np.float64) * self._fs
        out = np.zeros(m.ntot)
        for blk, elems in self.groups:
            idx = m.elem_idx[elems][:, m.loc_B]
            Y = u[idx] @ blk.Hhat.T
            out += np.bincount(idx.ravel(), weights=Y.ravel(), minlength=m.ntot)
        return out * self._fs

    def residual(self, u, f):
        """r_hat = F_hat - H_hat u_hat."""
        return (np.asarray(f) - self.apply(u)) * self._fs

    def diag(self):
        """diag(H_hat) assembled from the element Schur complements (Jacobi for coarse CG)."""
        m = self.mesh
        out = np.zeros(m.ntot)
        for blk, elems in self.groups:
            idx = m.elem_idx[elems][:, m.loc_B]
            d = np.tile(np.diag(blk.Hhat), (len(elems), 1))
            out += np.bincount(idx.ravel(), weights=d.ravel(), minlength=m.ntot)
        return out * self._fs

    def condense(self, F):
        """F_hat = F_B - H_BI H_II^-1 F_I (Alg. 4 line 2 / P:494)."""
        m = self.mesh
        F = np.asarray(F, dtype=np.float64) * self._free
        out = F * self._fs
        for blk, elems in self.groups:
            idxB = m.elem_idx[elems][:, m.loc_B]
            idxI = m.elem_idx[elems][:, m.loc_I]
            if idxI.shape[1] == 0:
                continue
            Z = blk.solve_II(F[idxI].T)          # (nI, ne)
            Y = (blk.HBI @ Z).T                  # (ne, nB)
            out -= np.bincount(idxB.ravel(), weights=Y.ravel(), minlength=m.ntot)
        return out * self._fs

    def recover(self, u_hat, F):
        """u = (u_hat, H_II^-1 (F_I - H_IB u_hat)) (Alg. 4 last line)."""
        m = self.mesh
        F = np.asarray(F, dtype=np.float64) * self._free
        u_hat = np.asarray(u_hat, dtype=np.float64) * self._fs
        u = u_hat.copy()
        for blk, elems in self.groups:
            idxB = m.elem_idx[elems][:, m.loc_B]
            idxI = m.elem_idx[elems][:, m.loc_I]
            if idxI.shape[1] == 0:
                continue
            rhs = F[idxI].T - blk.HIB @ u_hat[idxB].T
            u[idxI.ravel()] = blk.solve_II(rhs).T.ravel()
        return u * self._free

    # --- full (uncondensed) system, for brute-force checks ----------------------------
    def apply_full(self, u):
        m = self.mesh
        u = np.asarray(u, dtype=np.float64) * self._free
        out = np.zeros(m.ntot)
        for blk, elems in self.groups:
            idx = m.elem_idx[elems]
            Y = u[idx] @ blk.H.T
            out += np.bincount(idx.ravel(), weights=Y.ravel(), minlength=m.ntot)
        return out * self._free

    def assembled_full(self):
        """Sparse assembled H (all grid points; rows/cols of Dirichlet points kept)."""
        m = self.mesh
        rows, cols, vals = [], [], []
        for blk, elems in self.groups:
            idx = m.elem_idx[elems]
            n = idx.shape[1]
            rows.append(np.repeat(idx, n, axis=1).ravel())
            cols.append(np.tile(idx, (1, n)).ravel())
            vals.append(np.tile(blk.H.ravel(), len(elems)))
        return sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                             shape=(m.ntot, m.ntot)).tocsr()

    def assembled_condensed(self):
        """Sparse assembled H_hat = sum_e Q_hat_e H_hat_e Q_hat_e^T (all grid points)."""
        m = self.mesh
        rows, cols, vals = [], [], []
        for blk, elems in self.groups:
            idx = m.elem_idx[elems][:, m.loc_B]
            n = idx.shape[1]
            rows.append(np.repeat(idx, n, axis=1).ravel())
            cols.append(np.tile(idx, (1, n)).ravel())
            vals.append(np.tile(blk.Hhat.ravel(), len(elems)))
        return sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                             shape=(m.ntot, m.ntot)).tocsr()


def lumped_mass_1d(mesh, d):
    """Assembled 1-D GLL-lumped mass along direction d: b_d[i] = sum over 1-D elements
    containing node i of (h_e/2) w_t."""
    from .gll import gll
    _, w = gll(mesh.p)
    p = mesh.p
    b = np.zeros(mesh.N[d])
    for e in range(mesh.k[d]):
        b[e * p:(e + 1) * p + 1] += 0.5 * mesh.widths[d][e] * w
    if mesh.is_periodic(d):   # node k_d p is node 0
        b[0] += b[-1]
        b[-1] = b[0]
    return b


def weak_rhs(mesh, f_nodal):
    """F = B f: the assembled GLL-lumped mass times the nodal values of f (reading c-8).

    B is diagonal; B_ii = sum over elements containing node i of prod_d (h_d/2) w_{t_d}.  The
    set of elements containing a node is a Cartesian product of 1-D element sets, so this
    sum equals b1[i1] b2[i2] b3[i3] (checked against the element loop ``_weak_rhs_loop``)."""
    b = [lumped_mass_1d(mesh, d) for d in range(3)]
    B = (b[2][:, None, None] * b[1][None, :, None] * b[0][None, None, :]).ravel()
    return B * np.asarray(f_nodal, dtype=np.float64).ravel() * mesh.free


def _weak_rhs_loop(mesh, f_nodal):
    from .gll import gll
    _, w = gll(mesh.p)
    out = np.zeros(mesh.ntot)
    t1, t2, t3 = mesh.local_t
    for e in range(mesh.n_elements):
        h = mesh.elem_h[e]
        b = (0.5 * h[0] * w[t1]) * (0.5 * h[1] * w[t2]) * (0.5 * h[2] * w[t3])
        np.add.at(out, mesh.elem_idx[e], b)
    return out * np.asarray(f_nodal, dtype=np.float64).ravel() * mesh.free
