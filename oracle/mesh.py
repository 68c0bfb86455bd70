"""Structured Cartesian spectral-element mesh on the global GLL tensor grid (oracle).

P:65-74 (Sec. 2.1): nodal basis, global operator assembled from element operators,
H = sum_e Q_e H_e Q_e^T.  P:89-91: cuboidal elements with widths h_{i,e}.
Homogeneous Dirichlet conditions on the whole box boundary (BASELINE configs).

Global point (i1, i2, i3), 0 <= i_d <= k_d p, flat index g = i1 + N1 (i2 + N2 i3), x1 fastest.

Periodic directions ("in the periodic case the ghost elements stay
part of the domain, requiring no change in the operator"): the global index along d is taken
modulo k_d p, so element k_d - 1 couples to the nodes of element 0; the grid keeps N_d = k_d p + 1
nodes, and the last plane (i_d = k_d p) is a duplicate of plane 0 that carries no unknown.
"""
import numpy as np

from .gll import gll


class Mesh:
    def __init__(self, k, widths, p, origin=(0.0, 0.0, 0.0), neumann=0, periodic=0):
        """neumann: bit 2d / 2d+1 set = homogeneous Neumann on the low / high face of direction d
        (SURVEY 8(f) NEXT-3); every other face is homogeneous Dirichlet.
        periodic: bit d set = direction d is periodic (needs k_d >= 2, no Neumann bits on d)."""
        self.neumann = int(neumann)
        self.periodic = int(periodic)
        for d in range(3):
            if self.periodic >> d & 1:
                if self.neumann >> (2 * d) & 3:
                    raise ValueError("a periodic direction has no Neumann faces")
                if int(k[d]) < 2:
                    raise ValueError("a periodic direction needs k_d >= 2")
        self.k = tuple(int(v) for v in k)
        self.p = int(p)
        if self.p < 1:
            raise ValueError("p >= 1 required")
        self.widths = [np.asarray(w, dtype=np.float64).copy() for w in widths]
        for d in range(3):
            if len(self.widths[d]) != self.k[d]:
                raise ValueError("widths[%d] must have k_d entries" % d)
            if np.any(self.widths[d] <= 0) or not np.all(np.isfinite(self.widths[d])):
                raise ValueError("widths must be positive and finite")
        self.N = tuple(kd * self.p + 1 for kd in self.k)
        self.ntot = self.N[0] * self.N[1] * self.N[2]
        xi, _ = gll(self.p)
        # 1-D coordinates of the global GLL nodes per direction
        self.coords = []
        for d in range(3):
            x = np.zeros(self.N[d])
            x0 = origin[d]
            for e in range(self.k[d]):
                h = self.widths[d][e]
                x[e * self.p: (e + 1) * self.p + 1] = x0 + 0.5 * (xi + 1.0) * h
                x0 += h
            self.coords.append(x)
        i3, i2, i1 = np.meshgrid(np.arange(self.N[2]), np.arange(self.N[1]), np.arange(self.N[0]),
                                 indexing="ij")
        self.idx = (i1, i2, i3)
        interior = self.free1d(0, i1) & self.free1d(1, i2) & self.free1d(2, i3)
        skel = (i1 % self.p == 0) | (i2 % self.p == 0) | (i3 % self.p == 0)
        self.free = interior.ravel()              # not on a Dirichlet face
        self.skel = skel.ravel()                  # element-boundary points
        self.free_skel = self.free & self.skel    # condensed unknowns
        self._build_elements()

    def is_periodic(self, d):
        return bool(self.periodic >> d & 1)

    def wrap(self, d, g):
        """Global 1-D index along d as stored: modulo k_d p in a periodic direction."""
        g = np.asarray(g)
        return np.mod(g, self.k[d] * self.p) if self.is_periodic(d) else g

    def xcoord(self, d, g):
        """Coordinate of (possibly unwrapped) global 1-D index g: a periodic direction continues
        with the period (the box length) beyond its ends."""
        g = np.asarray(g)
        if not self.is_periodic(d):
            return self.coords[d][g]
        n = self.k[d] * self.p
        L = float(np.sum(self.widths[d]))
        return self.coords[d][np.mod(g, n)] + L * np.floor_divide(g, n)

    def fill_periodic(self, u):
        """Copy plane 0 of every periodic direction into its duplicate last plane (grid output)."""
        u = np.asarray(u, dtype=np.float64).reshape(self.N[2], self.N[1], self.N[0]).copy()
        if self.is_periodic(0):
            u[:, :, -1] = u[:, :, 0]
        if self.is_periodic(1):
            u[:, -1, :] = u[:, 0, :]
        if self.is_periodic(2):
            u[-1, :, :] = u[0, :, :]
        return u.ravel()

    def free1d(self, d, g):
        """Global 1-D indices g along d that are unknowns: inside [0, N_d - 1] and not on a
        Dirichlet end (a Neumann end point is an unknown); periodic: [0, N_d - 2] (the last index
        duplicates index 0)."""
        g = np.asarray(g)
        if self.is_periodic(d):
            return (g >= 0) & (g < self.N[d] - 1)
        lo = bool(self.neumann >> (2 * d) & 1)
        hi = bool(self.neumann >> (2 * d + 1) & 1)
        return (g >= 0) & (g <= self.N[d] - 1) & ((g > 0) | lo) & ((g < self.N[d] - 1) | hi)

    def flat(self, i1, i2, i3):
        return np.asarray(i1) + self.N[0] * (np.asarray(i2) + self.N[1] * np.asarray(i3))

    @property
    def n_elements(self):
        return self.k[0] * self.k[1] * self.k[2]

    def _build_elements(self):
        p = self.p
        t = np.arange(p + 1)
        t3, t2, t1 = np.meshgrid(t, t, t, indexing="ij")
        t1, t2, t3 = t1.ravel(), t2.ravel(), t3.ravel()   # local lexicographic, x1 fastest
        self.local_t = (t1, t2, t3)
        on_b = (t1 % p == 0) | (t2 % p == 0) | (t3 % p == 0)
        self.loc_B = np.nonzero(on_b)[0]
        self.loc_I = np.nonzero(~on_b)[0]
        elems, hs = [], []
        for e3 in range(self.k[2]):
            for e2 in range(self.k[1]):
                for e1 in range(self.k[0]):
                    elems.append(self.flat(self.wrap(0, e1 * p + t1), self.wrap(1, e2 * p + t2),
                                           self.wrap(2, e3 * p + t3)))
                    hs.append((self.widths[0][e1], self.widths[1][e2], self.widths[2][e3]))
        self.elem_idx = np.array(elems, dtype=np.int64)      # (n_e, (p+1)^3) global flat indices
        self.elem_h = np.array(hs, dtype=np.float64)          # (n_e, 3)

    def element_groups(self):
        """Elements grouped by their width triple (identical element operators)."""
        keys = {}
        for e, h in enumerate(self.elem_h):
            keys.setdefault(tuple(h.tolist()), []).append(e)
        return [(np.array(k), np.array(v, dtype=np.int64)) for k, v in keys.items()]

    def grid(self, v):
        return np.asarray(v).reshape(self.N[2], self.N[1], self.N[0])
