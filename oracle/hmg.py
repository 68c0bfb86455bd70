"""Low-order (h-)multigrid preconditioner for the p0 = 2 coarse level (oracle).

SURVEY 8(f) NEXT-2: the coarse solve costs O(n_e^alpha) with alpha = 4/3 for the CG
used in the paper; "alpha = 1 can be attained by reverting to an appropriate low-order multigrid
solver".  Reading R16: the coarse level keeps its conjugate-gradient iteration
and gains a symmetric h-multigrid V-cycle as preconditioner:

  - h-levels: the p = 2 condensed system on element-merged meshes: a direction is halved (pairs
    of elements merged, widths summed) while its k_d is even with k_d / 2 >= 2 (directions that
    cannot be halved keep their elements: semi-coarsening); levels continue while any direction
    halves and the current level has more than DENSE_MAX free unknowns;
  - transfer: P = fine free skeleton <- coarse free skeleton, the coarse element's quadratic
    (tensor GLL Lagrange basis on {-1, 0, 1}) evaluated at the fine nodes, with the coarse
    element's interior (centre) value given by its harmonic extension
    u_c = -H_cB u_B / H_cc (the static-condensation recovery with zero load);
    restriction R = P^T;
  - smoother: nu damped Jacobi sweeps x <- x + omega D^-1 (f - A x), omega = 0.6, before and after
    the coarse correction (symmetric V-cycle);
  - coarsest h-level (at most DENSE_MAX free unknowns): solved exactly (dense); larger coarsest
    levels: COARSEST_SWEEPS damped Jacobi sweeps from zero (a fixed symmetric operator).

Plain NumPy/SciPy, every step written out; test infrastructure only.
"""
import numpy as np
import scipy.sparse as sp

from .condensed import CondensedOperator, element_operator
from .gll import gll
from .mesh import Mesh

OMEGA = 0.6
NU = 2
COARSEST_SWEEPS = 40
DENSE_MAX = 1500


def halvable(kd):
    return kd % 2 == 0 and kd // 2 >= 2


def coarsenable(k):
    return any(halvable(kd) for kd in k)


def coarsen(k, widths):
    """(k_c, widths_c): every halvable direction merged pairwise, the others unchanged."""
    kc, wc = [], []
    for kd, w in zip(k, widths):
        w = np.asarray(w)
        if halvable(kd):
            kc.append(kd // 2)
            wc.append(w[0::2] + w[1::2])
        else:
            kc.append(kd)
            wc.append(w.copy())
    return tuple(kc), wc


def merged_widths(widths):
    return [np.asarray(w[0::2]) + np.asarray(w[1::2]) for w in widths]


def quad_basis(xi):
    """Lagrange basis on the p = 2 GLL nodes {-1, 0, 1} at xi."""
    return np.array([0.5 * xi * (xi - 1.0), 1.0 - xi * xi, 0.5 * xi * (xi + 1.0)])


def h_prolongation(mesh_c, mesh_f, lam):
    """Sparse P: fine free skeleton <- coarse free skeleton (ntot_f x ntot_c)."""
    p = 2
    t = np.arange(3)
    t3, t2, t1 = np.meshgrid(t, t, t, indexing="ij")
    t1, t2, t3 = t1.ravel(), t2.ravel(), t3.ravel()                 # local node order (x1 fastest)
    centre = 13                                                     # (1, 1, 1)
    rows, cols, vals = [], [], []
    cache = {}
    fs = np.nonzero(mesh_f.free_skel)[0]
    N1, N2 = mesh_f.N[0], mesh_f.N[1]
    for gf in fs:
        G = (gf % N1, (gf // N1) % N2, gf // (N1 * N2))
        ratio = [mesh_f.k[d] // mesh_c.k[d] for d in range(3)]          # 2 (merged) or 1 (kept)
        ec = [min(G[d] // (2 * ratio[d]), mesh_c.k[d] - 1) for d in range(3)]
        w = np.ones(27)
        for d in range(3):
            xa = mesh_c.coords[d][ec[d] * p]
            xb = mesh_c.coords[d][ec[d] * p + p]
            xi = 2.0 * (mesh_f.coords[d][G[d]] - xa) / (xb - xa) - 1.0
            w *= quad_basis(xi)[[t1, t2, t3][d]]
        h = tuple(mesh_c.widths[d][ec[d]] for d in range(3))
        if h not in cache:
            cache[h] = element_operator(p, h, lam)
        H = cache[h]
        wb = w + w[centre] * (-H[centre] / H[centre, centre])    # harmonic extension of the centre
        wb[centre] = 0.0
        gc = mesh_c.flat(ec[0] * p + t1, ec[1] * p + t2, ec[2] * p + t3)
        for i in range(27):
            if i == centre or wb[i] == 0.0 or not mesh_c.free_skel[gc[i]]:
                continue
            rows.append(gf)
            cols.append(gc[i])
            vals.append(wb[i])
    return sp.csr_matrix((vals, (rows, cols)), shape=(mesh_f.ntot, mesh_c.ntot))


class HLevel:
    def __init__(self, k, widths, lam, neumann):
        self.mesh = Mesh(k, widths, 2, neumann=neumann)
        self.op = CondensedOperator(self.mesh, lam)
        d = self.op.diag()
        self.dinv = np.where(d != 0, 1.0 / np.where(d != 0, d, 1.0), 0.0) * self.mesh.free_skel


class HMultigrid:
    """Symmetric h-multigrid V-cycle on the p = 2 condensed system (a linear operator M^-1)."""

    def __init__(self, k, widths, lam, neumann=0):
        self.levels = [HLevel(k, widths, lam, neumann)]
        # coarsen until a level is small enough for the exact (dense) coarsest solve
        while coarsenable(self.levels[-1].mesh.k) and int(self.levels[-1].mesh.free_skel.sum()) > DENSE_MAX:
            m = self.levels[-1].mesh
            kc, wc = coarsen(m.k, m.widths)
            self.levels.append(HLevel(kc, wc, lam, neumann))
        self.P = [h_prolongation(self.levels[l + 1].mesh, self.levels[l].mesh, lam)
                  for l in range(len(self.levels) - 1)]
        self.R = [P.T.tocsr() for P in self.P]

    def smooth(self, l, x, f, sweeps):
        lv = self.levels[l]
        for _ in range(sweeps):
            x = x + OMEGA * lv.dinv * (f - lv.op.apply(x))
        return x

    def vcycle(self, f, l=0):
        lv = self.levels[l]
        x = np.zeros(lv.mesh.ntot)
        if l == len(self.levels) - 1:
            fs = np.nonzero(lv.mesh.free_skel)[0]
            if len(fs) <= DENSE_MAX:
                A = lv.op.assembled_condensed()[fs][:, fs].toarray()
                x[fs] = np.linalg.solve(A, np.asarray(f)[fs])
                return x
            return self.smooth(l, x, f, COARSEST_SWEEPS)
        x = self.smooth(l, x, f, NU)
        r = (f - lv.op.apply(x)) * lv.mesh.free_skel
        x = x + self.P[l] @ self.vcycle(self.R[l] @ r, l + 1)
        return self.smooth(l, x, f, NU)


def pcg_hmg(level, hmg, b, rtol, maxit):
    """CG on the coarse condensed system with the h-multigrid V-cycle as preconditioner; stops at
    the first iteration with ||r|| <= rtol ||b|| (as mg.pcg)."""
    A = level.op
    b = np.asarray(b, dtype=np.float64) * level.mesh.free_skel
    x = np.zeros_like(b)
    r = b.copy()
    nb = float(np.sqrt(b @ b))
    if nb == 0.0:
        return x, 0
    z = hmg.vcycle(r)
    p = z.copy()
    rz = float(r @ z)
    for it in range(1, maxit + 1):
        q = A.apply(p)
        alpha = rz / float(p @ q)
        x = x + alpha * p
        r = r - alpha * q
        if np.sqrt(float(r @ r)) <= rtol * nb:
            return x, it
        z = hmg.vcycle(r)
        rz_new = float(r @ z)
        p = z + (rz_new / rz) * p
        rz = rz_new
    return x, maxit
