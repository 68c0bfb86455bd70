"""Element-centred block smoother (oracle).  TEST INFRASTRUCTURE ONLY: imported by tests/,
__graft_entry__.smoke() and bench.py's CPU legs, never by the product path.

SURVEY 8(f) NEXT-4, P:390-417 (Sec. "Extension to element-centered block smoothers"):
  - the subdomain of element e is the 3 x 3 x 3 element block centred on it ("full overlap",
    P:399-400), the one-dimensional matrices "replaced by those restricted to the subdomain"
    (P:401): three elements assembled, the block's outer end points dropped, so n_S = 3p - 1
    points per direction;
  - after condensation the unknowns of the block are the points of the SIX planes through the
    faces of the centre element (Fig. element_centered_block right): along direction d
    the local positions c_lo = p - 1 and c_hi = 2p - 1;
  - the block operator is the restriction of the condensed operator, H_i = R_i H_hat R_i^T
    (Eq. smoother_definition), and its inverse is applied through the fast
    diagonalisation of the full block with six faces instead of three: 73 n_S^3
    operations;
  - boundary blocks keep their shape; points outside the domain or on a Dirichlet face are
    decoupled (identity padding), Neumann faces stay unknowns (as the star);
  - weights (reading R17; the paper does not state them for this smoother): the
    tensor product of 1-D partitions of unity built from the star's weight polynomial w
    (P:312-316): omega_e(x) = (1/2) [ (1 + [e = 0]) w_{X_e}(x) + (1 + [e = k-1]) w_{X_{e+1}}(x) ],
    w_V(x) = w(|x - X_V| / h) on the two elements adjoining the vertex V (0 elsewhere).  On the
    centre element omega = 1/2, it falls to 0 at the block's outer ends, and
    sum_e omega_e = sum_V w_V = 1 along every grid line.

The oracle inverts every block by a DENSE LU factorisation of its explicitly assembled condensed
operator (``ec_matrix_block``); ``ec_matrix_schur`` eliminates the interiors of the assembled
uncondensed block; ``tpc_ec_inverse`` is the six-face fast-diagonalisation algorithm step by step
(the GPU kernel's arithmetic), checked here against the dense route.
"""
import numpy as np
import scipy.linalg as sla

from .gll import element_matrices_1d, weight_poly
from .smoother import _padded_fdm


def ec_n(p):
    return 3 * p - 1


def ec_planes(p):
    """Local positions of the centre element's two faces along a block line (0-based)."""
    return (p - 1, 2 * p - 1)


def ec_index_range(mesh, e, d):
    """Global 1-D indices of the n_S = 3p-1 block points along direction d for element e."""
    p = mesh.p
    return np.arange((e[d] - 1) * p + 1, (e[d] + 2) * p)


def ec_points(mesh, e):
    """Free block points of element e in canonical order (j3 slow, j1 fast over the n_S^3 cube,
    keeping the points on one of the six face planes).  Returns flat global indices and the local
    (j1, j2, j3) coordinates."""
    p = mesh.p
    n = ec_n(p)
    cl, ch = ec_planes(p)
    g = [ec_index_range(mesh, e, d) for d in range(3)]
    j3, j2, j1 = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    j1, j2, j3 = j1.ravel(), j2.ravel(), j3.ravel()
    on_plane = np.zeros(j1.shape, dtype=bool)
    for j in (j1, j2, j3):
        on_plane |= (j == cl) | (j == ch)
    G1, G2, G3 = g[0][j1], g[1][j2], g[2][j3]
    valid = mesh.free1d(0, G1) & mesh.free1d(1, G2) & mesh.free1d(2, G3)
    keep = on_plane & valid
    return mesh.flat(G1[keep], G2[keep], G3[keep]), (j1[keep], j2[keep], j3[keep])


def ec_weight_1d(mesh, e, d, g, pw=7):
    """omega_e along direction d at global 1-D indices g of the block line (reading R17)."""
    p, k = mesh.p, mesh.k[d]
    x = mesh.coords[d][np.clip(g, 0, mesh.N[d] - 1)]
    out = np.zeros(len(g))
    for V, mult in ((e[d], 2.0 if e[d] == 0 else 1.0), (e[d] + 1, 2.0 if e[d] == k - 1 else 1.0)):
        XV = mesh.coords[d][V * p]
        near = (g >= (V - 1) * p) & (g <= (V + 1) * p)
        side = np.where(g < V * p, V - 1, V)
        h = mesh.widths[d][np.clip(side, 0, k - 1)]
        t = np.abs(x - XV) / h
        out += np.where(near, 0.5 * mult * weight_poly(np.minimum(t, 1.0), pw), 0.0)
    return out


def ec_weights(mesh, e, loc, pw=7):
    W = np.ones(len(loc[0]))
    for d in range(3):
        W *= ec_weight_1d(mesh, e, d, ec_index_range(mesh, e, d)[loc[d]], pw)
    return W


def elements(mesh):
    out = []
    for e3 in range(mesh.k[2]):
        for e2 in range(mesh.k[1]):
            for e1 in range(mesh.k[0]):
                out.append((e1, e2, e3))
    return out


def ec_block_elements(mesh, e):
    """Elements of the 3x3x3 block around element e that exist in the mesh."""
    out = []
    for e3 in (e[2] - 1, e[2], e[2] + 1):
        for e2 in (e[1] - 1, e[1], e[1] + 1):
            for e1 in (e[0] - 1, e[0], e[0] + 1):
                if 0 <= e1 < mesh.k[0] and 0 <= e2 < mesh.k[1] and 0 <= e3 < mesh.k[2]:
                    out.append(e1 + mesh.k[0] * (e2 + mesh.k[1] * e3))
    return out


def ec_matrix_block(condop, e, pts):
    """H_i = R_i H_hat R_i^T assembled from the Schur complements of the 27 block elements."""
    mesh = condop.mesh
    pos = {int(g): i for i, g in enumerate(pts)}
    H = np.zeros((len(pts), len(pts)))
    blk_of = {}
    for blk, elems in condop.groups:
        for el in elems:
            blk_of[int(el)] = blk
    for el in ec_block_elements(mesh, e):
        gB = mesh.elem_idx[el][mesh.loc_B]
        sel = [i for i, g in enumerate(gB) if int(g) in pos]
        tgt = [pos[int(gB[i])] for i in sel]
        H[np.ix_(tgt, tgt)] += blk_of[el].Hhat[np.ix_(sel, sel)]
    return H


def ec_1d(mesh, e, d):
    """1-D mass/stiffness of the block line along d: the three elements e-1, e, e+1
    (those in the mesh) assembled, the outer end points dropped (n_S = 3p-1), plus the mask of
    points inside the domain and off the Dirichlet boundary."""
    p = mesh.p
    n = ec_n(p)
    M = np.zeros((n, n))
    K = np.zeros((n, n))
    for side in range(3):
        el = e[d] - 1 + side
        if not (0 <= el < mesh.k[d]):
            continue
        Me, Ke = element_matrices_1d(p, mesh.widths[d][el])
        for t in range(p + 1):
            j = side * p - 1 + t
            if not (0 <= j < n):
                continue
            for s in range(p + 1):
                i = side * p - 1 + s
                if 0 <= i < n:
                    K[j, i] += Ke[t, s]
            M[j, j] += Me[t, t]
    valid = mesh.free1d(d, ec_index_range(mesh, e, d))
    return M, K, valid


def ec_matrix_schur(condop, e, loc):
    """Schur complement of the assembled uncondensed block operator (tensor form) onto
    the free plane points given by local coords ``loc`` (interiors of the 27 elements
    eliminated)."""
    mesh = condop.mesh
    lam = condop.lam
    n = ec_n(mesh.p)
    cl, ch = ec_planes(mesh.p)
    (M1, K1, v1), (M2, K2, v2), (M3, K3, v3) = [ec_1d(mesh, e, d) for d in range(3)]
    H = (lam * np.kron(M3, np.kron(M2, M1)) + np.kron(M3, np.kron(M2, K1))
         + np.kron(M3, np.kron(K2, M1)) + np.kron(K3, np.kron(M2, M1)))
    j3, j2, j1 = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    j1, j2, j3 = j1.ravel(), j2.ravel(), j3.ravel()
    valid = v1[j1] & v2[j2] & v3[j3]
    on_plane = np.zeros(j1.shape, dtype=bool)
    for j in (j1, j2, j3):
        on_plane |= (j == cl) | (j == ch)
    S = np.nonzero(valid & on_plane)[0]
    I = np.nonzero(valid & ~on_plane)[0]
    Hc = H[np.ix_(S, S)] - H[np.ix_(S, I)] @ np.linalg.solve(H[np.ix_(I, I)], H[np.ix_(I, S)])
    flatS = j1[S] + n * (j2[S] + n * j3[S])
    want = loc[0] + n * (loc[1] + n * loc[2])
    perm = np.searchsorted(flatS, want)
    assert np.array_equal(flatS[perm], want)
    return Hc[np.ix_(perm, perm)]


def tpc_ec_inverse(condop, e, r):
    """The six-face fast-diagonalisation inverse, step by step:
      1. per face plane (d, c): F_{d,c}[A, B] = r on the plane / (number of planes through the
         point) -- every plane point is stored once per plane it lies on;
      2. F_E = sum_{d, c} S_d[c, :] (x) S_d'^T (x) S_d''^T F_{d,c}   (eigenspace right-hand side
         of the full block with zero interiors);
      3. U_E = F_E / (lambda + Lambda_1 + Lambda_2 + Lambda_3);
      4. U_{d,c} = S_d[c, :] (x) S_d' (x) S_d'' U_E on each plane (the block solution there).
    Returns the solution on the free block points in ``ec_points`` order."""
    mesh = condop.mesh
    lam = condop.lam
    p = mesh.p
    n = ec_n(p)
    cl, ch = ec_planes(p)
    pts, loc = ec_points(mesh, e)
    SL, va = [], []
    for d in range(3):
        M, K, valid = ec_1d(mesh, e, d)
        SL.append(_padded_fdm(M, K, valid))
        va.append(valid)
    (S1, L1), (S2, L2), (S3, L3) = SL
    g = [ec_index_range(mesh, e, d) for d in range(3)]
    R = np.asarray(r)
    jj = np.arange(n)
    A, B = np.meshgrid(jj, jj, indexing="ij")            # A = slow index, B = fast index

    def val(i1, i2, i3, ok):
        out = np.zeros(i1.shape)
        out[ok] = R[mesh.flat(i1[ok], i2[ok], i3[ok])]
        return out

    def nplanes(a, b):
        return 1 + ((a == cl) | (a == ch)) + ((b == cl) | (b == ch))

    FE = np.zeros((n, n, n))                              # [a3, a2, a1]
    faces = {}
    for c in (cl, ch):
        F1 = val(np.full_like(A, g[0][c]), g[1][B], g[2][A], va[0][c] & va[1][B] & va[2][A]) / nplanes(A, B)
        F2 = val(g[0][B], np.full_like(A, g[1][c]), g[2][A], va[0][B] & va[1][c] & va[2][A]) / nplanes(A, B)
        F3 = val(g[0][B], g[1][A], np.full_like(A, g[2][c]), va[0][B] & va[1][A] & va[2][c]) / nplanes(A, B)
        FE += np.einsum("a,xc,yb,xy->cba", S1[c, :], S3, S2, F1)   # plane j1 = c: F1[j3, j2]
        FE += np.einsum("b,xc,ya,xy->cba", S2[c, :], S3, S1, F2)   # plane j2 = c: F2[j3, j1]
        FE += np.einsum("c,xb,ya,xy->cba", S3[c, :], S2, S1, F3)   # plane j3 = c: F3[j2, j1]
    UE = FE / (lam + L1[None, None, :] + L2[None, :, None] + L3[:, None, None])
    for c in (cl, ch):
        faces[(0, c)] = np.einsum("a,xc,yb,cba->xy", S1[c, :], S3, S2, UE)   # [j3, j2]
        faces[(1, c)] = np.einsum("b,xc,ya,cba->xy", S2[c, :], S3, S1, UE)   # [j3, j1]
        faces[(2, c)] = np.einsum("c,xb,ya,cba->xy", S3[c, :], S2, S1, UE)   # [j2, j1]
    j1, j2, j3 = loc
    out = np.empty(len(pts))
    for i in range(len(pts)):
        a, b, cc = j1[i], j2[i], j3[i]
        if a in (cl, ch):
            out[i] = faces[(0, a)][cc, b]
        elif b in (cl, ch):
            out[i] = faces[(1, b)][cc, a]
        else:
            out[i] = faces[(2, cc)][b, a]
    return pts, out


class ECSmoother:
    """Eq. (smoother_definition) over the element-centred blocks, dense-LU block inverses cached
    per block shape (identical widths of the three elements per direction)."""

    def __init__(self, condop, pw=7):
        self.condop = condop
        mesh = condop.mesh
        self.mesh = mesh
        classes = {}
        for e in elements(mesh):
            key = []
            for d in range(3):
                key.append(tuple(mesh.widths[d][x] if 0 <= x < mesh.k[d] else None
                                 for x in (e[d] - 1, e[d], e[d] + 1)))
            classes.setdefault(tuple(key), []).append(e)
        self.classes = []
        for key, members in classes.items():
            pts0, loc0 = ec_points(mesh, members[0])
            if len(pts0) == 0:
                continue
            lu = sla.lu_factor(ec_matrix_block(condop, members[0], pts0))
            W = ec_weights(mesh, members[0], loc0, pw)
            P = np.stack([ec_points(mesh, e)[0] for e in members])
            self.classes.append((lu, W, P, members))

    @property
    def n_blocks(self):
        return sum(len(c[3]) for c in self.classes)

    def apply(self, r):
        """du = sum_i R_i^T W_i H_i^-1 R_i r."""
        mesh = self.mesh
        r = np.asarray(r, dtype=np.float64)
        du = np.zeros(mesh.ntot)
        for lu, W, P, _ in self.classes:
            X = sla.lu_solve(lu, r[P].T)
            du += np.bincount(P.ravel(), weights=(W[:, None] * X).T.ravel(), minlength=mesh.ntot)
        return du * mesh.free_skel
