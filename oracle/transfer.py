"""p-prolongation and restriction between condensed levels (oracle).

P:439 (Sec. 4.1): "The prolongation from level l-1 to level l, J_hat_l, is the embedded
interpolation, restricted from the tensor-product of one-dimensional prolongation operators to
the condensed system, and the restriction operator is its transpose."

Here J_hat = R_f (J (x) J (x) J) E_c: coarse skeleton values are extended by zero element
interiors (E_c), interpolated element by element with the tensor product of the 1-D matrix
J[i, a] = l_a^{coarse}(xi_i^{fine}), and restricted to the fine free skeleton (R_f).  A fine
point shared by several elements takes its value from one of them (all give the same value:
the endpoint rows of J are unit vectors).  The restriction is the explicit sparse transpose.
"""
import numpy as np
import scipy.sparse as sp

from .gll import interpolation_matrix


def prolongation_matrix(mesh_c, mesh_f):
    if mesh_c.k != mesh_f.k:
        raise ValueError("levels must share the element mesh")
    J = interpolation_matrix(mesh_c.p, mesh_f.p)
    P = np.kron(J, np.kron(J, J))                      # local (fine (p_f+1)^3) x (coarse (p_c+1)^3)
    Pb = P[np.ix_(mesh_f.loc_B, mesh_c.loc_B)]         # E_c: coarse interiors are zero
    rl, cl = np.nonzero(Pb)
    vals = Pb[rl, cl]
    ne = mesh_f.n_elements
    owner = np.full(mesh_f.ntot, -1, dtype=np.int64)
    for e in range(ne - 1, -1, -1):
        owner[mesh_f.elem_idx[e]] = e
    fB = mesh_f.elem_idx[:, mesh_f.loc_B]              # (ne, nBf)
    cB = mesh_c.elem_idx[:, mesh_c.loc_B]
    rows = fB[:, rl]                                   # (ne, nnz)
    cols = cB[:, cl]
    keep = (owner[rows] == np.arange(ne)[:, None]) & mesh_f.free_skel[rows] & mesh_c.free_skel[cols]
    data = np.broadcast_to(vals, rows.shape)[keep]
    return sp.csr_matrix((data, (rows[keep], cols[keep])), shape=(mesh_f.ntot, mesh_c.ntot))


class Transfer:
    def __init__(self, mesh_c, mesh_f):
        self.J = prolongation_matrix(mesh_c, mesh_f)
        self.JT = self.J.T.tocsr()

    def prolong(self, u_c):
        """J_hat_l u_{l-1} (fine free skeleton)."""
        return self.J @ np.asarray(u_c, dtype=np.float64)

    def restrict(self, r_f):
        """J_hat_l^T r_l (coarse free skeleton)."""
        return self.JT @ np.asarray(r_f, dtype=np.float64)
