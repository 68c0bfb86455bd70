"""Vertex-star additive Schwarz smoother (oracle).

P:126-149 Eq. (smoother_definition): du = sum_i R_i^T W_i H_i^-1 R_i r, H_i = R_i H R_i^T.
P:151-163: the subdomain of vertex i is the 2x2x2 element block around it; after
  condensation three planes of n_S x n_S points remain, n_S = 2p - 1 (block boundary dropped).
P:309-333 Alg. 2: loop over all vertex stars, extract, invert, weight and add.
P:312-316: W_i is the restriction of w(x)w(x)w with w the degree-7 weight polynomial.
P:348-375 Sec. 3.3: boundary vertices keep the same star shape; points outside the domain or
  on a Dirichlet face are decoupled (identity padding) and receive no correction; points on a
  Neumann face are unknowns of the star (NEXT-3).

The oracle inverts every star by a DENSE LU factorisation of its explicitly assembled condensed
operator (the north-star oracle; "matrix inversion").  ``star_matrix_block`` builds
H_i from the element Schur complements of the 8 block elements; ``star_matrix_global`` slices
it out of the assembled global H_hat (literally R_i H_hat R_i^T, small meshes only);
``star_matrix_schur`` eliminates the interiors of the assembled uncondensed block (Sec. 3.1).
``tpc_star_inverse`` follows Alg. 1 line by line and ``tpf_star_inverse`` applies Eq.
(fast_diagonalization) to the embedded right-hand side (Eq. star_right_hand_side_full); both
exist only to be checked against the dense LU route.
"""
import numpy as np
import scipy.linalg as sla

from .gll import gll, element_matrices_1d, weight_poly


def star_index_range(mesh, v, d):
    """Global 1-D indices of the n_S = 2p-1 star points along direction d for vertex v."""
    p = mesh.p
    return np.arange((v[d] - 1) * p + 1, (v[d] + 1) * p)


def star_points(mesh, v):
    """Free star points of vertex v in canonical order (j3 slow, j1 fast over the n_S^3 cube,
    keeping points on one of the three planes through the vertex).  Returns flat global
    indices and the local (j1, j2, j3) coordinates."""
    p = mesh.p
    n = 2 * p - 1
    c = p - 1
    g = [star_index_range(mesh, v, d) for d in range(3)]
    j3, j2, j1 = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    j1, j2, j3 = j1.ravel(), j2.ravel(), j3.ravel()
    on_plane = (j1 == c) | (j2 == c) | (j3 == c)
    G1, G2, G3 = mesh.wrap(0, g[0][j1]), mesh.wrap(1, g[1][j2]), mesh.wrap(2, g[2][j3])   # periodic: wrapped
    valid = mesh.free1d(0, G1) & mesh.free1d(1, G2) & mesh.free1d(2, G3)
    keep = on_plane & valid
    return mesh.flat(G1[keep], G2[keep], G3[keep]), (j1[keep], j2[keep], j3[keep])


def star_weights(mesh, v, loc, pw=7):
    """W_i at the star points: prod_d w(t_d), t_d = |x_d - x_d(vertex)| / h_d of the element
    containing the point on that side of the vertex (reading c-5: w is a polynomial of the
    coordinate on each of the two adjoining elements, Fig. weights)."""
    p = mesh.p
    W = np.ones(len(loc[0]))
    for d in range(3):
        g = star_index_range(mesh, v, d)[loc[d]]
        xv = mesh.coords[d][v[d] * p]
        e = np.where(g < v[d] * p, v[d] - 1, v[d])
        e = np.mod(e, mesh.k[d]) if mesh.is_periodic(d) else np.clip(e, 0, mesh.k[d] - 1)
        h = mesh.widths[d][e]
        t = np.abs(mesh.xcoord(d, g) - xv) / h
        W *= weight_poly(t, pw)
    return W


def vertices(mesh):
    """All mesh vertices ("the n_V vertices"), reading c-6: boundary vertices included; in a
    periodic direction vertex k_d is vertex 0."""
    n = [mesh.k[d] + (0 if mesh.is_periodic(d) else 1) for d in range(3)]
    out = []
    for v3 in range(n[2]):
        for v2 in range(n[1]):
            for v1 in range(n[0]):
                out.append((v1, v2, v3))
    return out


def block_elements(mesh, v):
    """Elements of the 2x2x2 block around vertex v that exist in the mesh."""
    out = []
    w = lambda d, e: e % mesh.k[d] if mesh.is_periodic(d) else e
    for e3 in (w(2, v[2] - 1), w(2, v[2])):
        for e2 in (w(1, v[1] - 1), w(1, v[1])):
            for e1 in (w(0, v[0] - 1), w(0, v[0])):
                if 0 <= e1 < mesh.k[0] and 0 <= e2 < mesh.k[1] and 0 <= e3 < mesh.k[2]:
                    out.append(e1 + mesh.k[0] * (e2 + mesh.k[1] * e3))
    return out


def star_matrix_block(condop, v, pts):
    """H_i = R_i H_hat R_i^T assembled from the Schur complements of the block elements."""
    mesh = condop.mesh
    pos = {int(g): i for i, g in enumerate(pts)}
    H = np.zeros((len(pts), len(pts)))
    blk_of = {}
    for blk, elems in condop.groups:
        for e in elems:
            blk_of[int(e)] = blk
    for e in block_elements(mesh, v):
        gB = mesh.elem_idx[e][mesh.loc_B]
        sel = [i for i, g in enumerate(gB) if int(g) in pos]
        tgt = [pos[int(gB[i])] for i in sel]
        H[np.ix_(tgt, tgt)] += blk_of[e].Hhat[np.ix_(sel, sel)]
    return H


def star_matrix_global(Hs_assembled, pts):
    """Literal R_i H_hat R_i^T from the assembled sparse condensed operator."""
    return Hs_assembled[pts][:, pts].toarray()


def star_1d(mesh, v, d):
    """1-D mass/stiffness matrices of the full star along d: assembled from the two
    elements adjoining the vertex, outer end points dropped (n_S = 2p-1), plus the mask of
    points inside the domain and off the Dirichlet boundary."""
    p = mesh.p
    n = 2 * p - 1
    M = np.zeros((n, n))
    K = np.zeros((n, n))
    for side, e in ((0, v[d] - 1), (1, v[d])):
        if mesh.is_periodic(d):
            e = e % mesh.k[d]
        if not (0 <= e < mesh.k[d]):
            continue
        Me, Ke = element_matrices_1d(p, mesh.widths[d][e])
        # element-local t = 0..p maps to star j = side*p - 1 + t ... restricted to 0..n-1
        for t in range(p + 1):
            j = side * p - 1 + t
            if not (0 <= j < n):
                continue
            for s in range(p + 1):
                i = side * p - 1 + s
                if 0 <= i < n:
                    K[j, i] += Ke[t, s]
            M[j, j] += Me[t, t]
    g = mesh.wrap(d, star_index_range(mesh, v, d))
    valid = mesh.free1d(d, g)
    return M, K, valid


def star_matrix_schur(condop, v, loc):
    """Schur complement of the assembled uncondensed block operator (Eq. helmholtzopstar,
    restricted to valid points) onto the free star points given by local coords ``loc``."""
    mesh = condop.mesh
    lam = condop.lam
    n = 2 * mesh.p - 1
    c = mesh.p - 1
    mats = [star_1d(mesh, v, d) for d in range(3)]
    M1, K1, v1 = mats[0]
    M2, K2, v2 = mats[1]
    M3, K3, v3 = mats[2]
    H = (lam * np.kron(M3, np.kron(M2, M1)) + np.kron(M3, np.kron(M2, K1))
         + np.kron(M3, np.kron(K2, M1)) + np.kron(K3, np.kron(M2, M1)))
    j3, j2, j1 = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    j1, j2, j3 = j1.ravel(), j2.ravel(), j3.ravel()
    valid = v1[j1] & v2[j2] & v3[j3]
    on_plane = (j1 == c) | (j2 == c) | (j3 == c)
    S = np.nonzero(valid & on_plane)[0]
    I = np.nonzero(valid & ~on_plane)[0]
    HSS = H[np.ix_(S, S)]
    HSI = H[np.ix_(S, I)]
    HII = H[np.ix_(I, I)]
    Hc = HSS - HSI @ np.linalg.solve(HII, HSI.T)
    # reorder to the order of ``loc``
    flatS = j1[S] + n * (j2[S] + n * j3[S])
    want = loc[0] + n * (loc[1] + n * loc[2])
    perm = np.searchsorted(flatS, want)
    assert np.array_equal(flatS[perm], want)
    return Hc[np.ix_(perm, perm)]


def _padded_fdm(M, K, valid):
    """Generalised eigenpairs S^T K S = Lambda, S^T M S = I on the coupled points, padded with
    identity on the decoupled ones."""
    n = len(valid)
    S = np.eye(n)
    L = np.ones(n)
    idx = np.nonzero(valid)[0]
    if len(idx):
        lam, Sc = sla.eigh(K[np.ix_(idx, idx)], M[np.ix_(idx, idx)])
        S[np.ix_(idx, idx)] = Sc
        L[idx] = lam
    return S, L


def tpc_star_inverse(condop, v, r):
    """Alg. 1, literally, with full n_S^3 eigenspace arrays.  Returns the star
    solution u~ on the free star points of ``star_points(mesh, v)`` order."""
    mesh = condop.mesh
    lam = condop.lam
    p = mesh.p
    n = 2 * p - 1
    c = p - 1
    pts, loc = star_points(mesh, v)
    fd = []
    for d in range(3):
        M, K, valid = star_1d(mesh, v, d)
        fd.append((_padded_fdm(M, K, valid), valid))
    (S1, L1), va1 = fd[0]
    (S2, L2), va2 = fd[1]
    (S3, L3), va3 = fd[2]
    g = [mesh.wrap(d, star_index_range(mesh, v, d)) for d in range(3)]
    R = np.asarray(r)

    def val(i1, i2, i3, ok):
        out = np.zeros(i1.shape)
        out[ok] = R[mesh.flat(i1[ok], i2[ok], i3[ok])]
        return out

    jj = np.arange(n)
    # face arrays: F1[j3, j2] at j1 = c ; F2[j3, j1] at j2 = c ; F3[j2, j1] at j3 = c
    A, B = np.meshgrid(jj, jj, indexing="ij")           # A = slow index, B = fast index
    F1 = val(np.full_like(A, g[0][c]), g[1][B], g[2][A], va1[c] & va2[B] & va3[A])
    F2 = val(g[0][B], np.full_like(A, g[1][c]), g[2][A], va1[B] & va2[c] & va3[A])
    F3 = val(g[0][B], g[1][A], np.full_like(A, g[2][c]), va1[B] & va2[A] & va3[c])
    # inverse multiplicity: a face point also lying on another plane is stored twice
    F1 = F1 / (1 + (A == c) + (B == c))
    F2 = F2 / (1 + (A == c) + (B == c))
    F3 = F3 / (1 + (A == c) + (B == c))
    s1, s2, s3 = S1[c, :], S2[c, :], S3[c, :]            # S_{I0}^T: row of S at the vertex
    # F_E = (S^T (x) S^T (x) S_I0^T) F1 + (S^T (x) S_I0^T (x) S^T) F2 + (S_I0^T (x) S^T (x) S^T) F3
    FE = np.zeros((n, n, n))                              # indices [a3, a2, a1]
    FE += np.einsum("a,xc,yb,xy->cba", s1, S3, S2, F1)    # a1 <- s1, a3 <- S3, a2 <- S2
    FE += np.einsum("b,xc,ya,xy->cba", s2, S3, S1, F2)    # a2 <- s2, a3 <- S3, a1 <- S1
    FE += np.einsum("c,xb,ya,xy->cba", s3, S2, S1, F3)    # a3 <- s3, a2 <- S2, a1 <- S1
    D = lam + L1[None, None, :] + L2[None, :, None] + L3[:, None, None]
    UE = FE / D
    U1 = np.einsum("a,xc,yb,cba->xy", s1, S3, S2, UE)     # U1[j3, j2]
    U2 = np.einsum("b,xc,ya,cba->xy", s2, S3, S1, UE)     # U2[j3, j1]
    U3 = np.einsum("c,xb,ya,cba->xy", s3, S2, S1, UE)     # U3[j2, j1]
    j1, j2, j3 = loc
    out = np.where(j1 == c, U1[j3, j2], np.where(j2 == c, U2[j3, j1], U3[j2, j1]))
    return pts, out


def tpf_star_inverse(condop, v, r):
    """Eq. (fast_diagonalization) applied to the embedded RHS (zero interior, Eq.
    star_right_hand_side_full), restricted back to the star planes (Sec. 3.1)."""
    mesh = condop.mesh
    lam = condop.lam
    p = mesh.p
    n = 2 * p - 1
    c = p - 1
    pts, loc = star_points(mesh, v)
    SL = []
    for d in range(3):
        M, K, valid = star_1d(mesh, v, d)
        SL.append(_padded_fdm(M, K, valid))
    (S1, L1), (S2, L2), (S3, L3) = SL
    Ft = np.zeros((n, n, n))
    Ft[loc[2], loc[1], loc[0]] = np.asarray(r)[pts]
    FE = np.einsum("xc,yb,za,xyz->cba", S3, S2, S1, Ft)
    D = lam + L1[None, None, :] + L2[None, :, None] + L3[:, None, None]
    U = np.einsum("xc,yb,za,cba->xyz", S3, S2, S1, FE / D)
    return pts, U[loc[2], loc[1], loc[0]]


class StarSmoother:
    """Alg. 2 with dense-LU star inverses, cached per star shape (identical block geometry)."""

    def __init__(self, condop, pw=7):
        self.condop = condop
        mesh = condop.mesh
        self.mesh = mesh
        classes = {}
        for v in vertices(mesh):
            key = []
            for d in range(3):
                if mesh.is_periodic(d):
                    key.append((mesh.widths[d][(v[d] - 1) % mesh.k[d]], mesh.widths[d][v[d]], "per"))
                    continue
                hl = mesh.widths[d][v[d] - 1] if v[d] >= 1 else None
                hr = mesh.widths[d][v[d]] if v[d] < mesh.k[d] else None
                key.append((hl, hr))
            classes.setdefault(tuple(key), []).append(v)
        self.classes = []
        for key, members in classes.items():
            pts0, loc0 = star_points(mesh, members[0])
            if len(pts0) == 0:
                continue                       # box corners: no free star point
            H = star_matrix_block(condop, members[0], pts0)
            lu = sla.lu_factor(H)
            W = star_weights(mesh, members[0], loc0, pw)
            P = np.stack([star_points(mesh, v)[0] for v in members])   # (nm, npts)
            self.classes.append((lu, W, P, members))

    @property
    def n_stars(self):
        return sum(len(c[3]) for c in self.classes)

    def apply(self, r):
        """du = sum_i R_i^T W_i H_i^-1 R_i r (Alg. 2 / Eq. smoother_definition)."""
        mesh = self.mesh
        r = np.asarray(r, dtype=np.float64)
        du = np.zeros(mesh.ntot)
        for lu, W, P, _ in self.classes:
            X = sla.lu_solve(lu, r[P].T)           # (npts, nm)
            Y = (W[:, None] * X).T
            du += np.bincount(P.ravel(), weights=Y.ravel(), minlength=mesh.ntot)
        return du * mesh.free_skel
