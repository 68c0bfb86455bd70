"""Full-size checks at the BASELINE.json configurations, in the launch configuration bench.py
times (the same Solver / pmg_solve path).  The oracle cannot hold these meshes, so outputs are
checked (a) one by one at sampled points, with the oracle's dense operators built on the small
sub-mesh that determines each sampled value (element operators depend only on the element widths;
the star inverse of an interior vertex is the inverse of the condensed operator of its 2x2x2 block
with a Dirichlet outer boundary, tests/test_oracle_star.py), and (b) through properties that hold at
any size (convergence to the 1e-10 drop, symmetry, the manufactured solution)."""
import math

import numpy as np
import pytest

import pmg_inputs as pi

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _solver(case, **kw):
    import paper_1808_03595_b200 as pmg
    return pmg.Solver(case.k, case.widths, case.p, case.lam, **kw)


def _grid_of(s, level, skel):
    g = s.new_grid(level)
    s.skel_to_grid(level, skel, g)
    torch.cuda.synchronize()
    return g.cpu().numpy()


class GridView:
    """Index helper on the global GLL grid of one level (no oracle arithmetic)."""

    def __init__(self, k, p):
        self.k, self.p = k, p
        self.N = tuple(kd * p + 1 for kd in k)

    def flat(self, i1, i2, i3):
        return i1 + self.N[0] * (i2 + self.N[1] * i3)


def _submesh(case, lo, n):
    """Mesh of n[0] x n[1] x n[2] elements starting at element lo, same widths, Dirichlet outside."""
    from oracle import mesh
    w = [case.widths[d][lo[d]:lo[d] + n[d]] for d in range(3)]
    return mesh.Mesh(n, w, case.p)


def _sampled_residual(case, ug, fg, rg, samples):
    """r at sampled skeleton points = f - sum over the elements containing the point of H_hat_e u_e."""
    from oracle import condensed
    p, k = case.p, case.k
    V = GridView(k, p)
    errs = []
    cache = {}
    for (i1, i2, i3) in samples:
        want = fg[V.flat(i1, i2, i3)]
        for e3 in {max(0, (i3 - 1) // p), min(k[2] - 1, i3 // p)}:
            for e2 in {max(0, (i2 - 1) // p), min(k[1] - 1, i2 // p)}:
                for e1 in {max(0, (i1 - 1) // p), min(k[0] - 1, i1 // p)}:
                    if not (e1 * p <= i1 <= (e1 + 1) * p and e2 * p <= i2 <= (e2 + 1) * p and e3 * p <= i3 <= (e3 + 1) * p):
                        continue
                    sub = _submesh(case, (e1, e2, e3), (1, 1, 1))
                    key = tuple(sub.elem_h[0].tolist())
                    if key not in cache:
                        cache[key] = condensed.ElementBlocks(p, sub.elem_h[0], case.lam, sub.loc_B, sub.loc_I)
                    blk = cache[key]
                    t1, t2, t3 = sub.local_t
                    gidx = V.flat(e1 * p + t1, e2 * p + t2, e3 * p + t3)[sub.loc_B]
                    ue = ug[gidx]
                    row = [j for j, (a, b, c) in enumerate(zip(t1[sub.loc_B], t2[sub.loc_B], t3[sub.loc_B]))
                           if (e1 * p + a, e2 * p + b, e3 * p + c) == (i1, i2, i3)][0]
                    want -= blk.Hhat[row] @ ue
        errs.append(abs(rg[V.flat(i1, i2, i3)] - want) / max(abs(want), np.abs(fg).max() * 1e-3))
    return max(errs)


def _interior_points(case, rng, nsample):
    p, k = case.p, case.k
    pts = []
    while len(pts) < nsample:
        v = [int(rng.integers(1, kd)) for kd in k]
        kind = len(pts) % 3
        i = [vd * p for vd in v]
        if kind >= 1:
            i[0] += int(rng.integers(1, p))          # edge point (x1 edge)
        if kind == 2:
            i[1] += int(rng.integers(1, p))          # face point (x3 face)
        pts.append(tuple(i))
    return pts


@pytest.mark.parametrize("cfg,p", [(2, None), (3, 2), (3, 4), (3, 8), (3, 12), (3, 16), (3, 24), (4, None)])
def test_fullsize_residual_sampled(cfg, p):
    """Bench-size residual at sampled vertex / edge / face points against the oracle's dense element
    Schur complements (p = 32 is compared element-wise on the small k222_p32 parity mesh instead: the
    same kernel, k_elem_apply_t<32>)."""
    case = pi.config(cfg, p=p)
    s = _solver(case)
    L = s.nlevels - 1
    rng = np.random.default_rng(cfg * 100 + (p or 0))
    n = s.level_info(L)[1]
    u = torch.from_numpy(rng.standard_normal(n)).cuda()
    f = torch.from_numpy(rng.standard_normal(n)).cuda()
    # normalise to free-skeleton vectors through the grid (zero on non-free entries)
    ugr, fgr = _grid_of(s, L, u), _grid_of(s, L, f)
    uu, ff = s.new_skel(L), s.new_skel(L)
    s.skel_from_grid(L, torch.from_numpy(ugr).cuda(), uu)
    s.skel_from_grid(L, torch.from_numpy(fgr).cuda(), ff)
    r = s.new_skel(L)
    s.residual(L, uu, ff, r)
    rgr = _grid_of(s, L, r)
    err = _sampled_residual(case, ugr, fgr, rgr, _interior_points(case, rng, 6))
    assert err < 1e-11, err
    # symmetry of the full-size operator
    a, b = s.new_skel(L), s.new_skel(L)
    s.residual(L, uu, None, a)
    s.residual(L, ff, None, b)
    x, y = float((a * ff).sum()), float((uu * b).sum())
    assert abs(x - y) <= 1e-11 * max(abs(x), 1.0)
    s.close()


def _sampled_smoother(case, rg, dug, rng, nsample):
    """Smoother correction at sampled interior skeleton points (vertex, edge-interior and
    face-interior points, in turn): sum over the stars whose planes contain the point of
    W_v(x) (H_hat_v^-1 R_v r)(x) (Eq. smoother_definition).  Each star inverse is the
    dense solve of the oracle's assembled condensed star operator on the 2x2x2-element sub-mesh
    around v (the block sees nothing else; Dirichlet outside is the block's own boundary),
    and W_v is the oracle's weight at the point.  A vertex is covered by its own star only (W = 1),
    an edge point by 2 stars, a face point by 4 (the weighted multi-star sum)."""
    from oracle import condensed, smoother
    p, k = case.p, case.k
    V = GridView(k, p)
    errs = []
    blocks = {}
    for i in range(nsample):
        kind = i % 3
        x = [int(rng.integers(2, kd - 1)) * p for kd in k]          # an interior vertex, one element from the box
        if kind >= 1:
            x[0] += int(rng.integers(1, p))                          # edge along x1
        if kind == 2:
            x[1] += int(rng.integers(1, p))                          # face normal to x3
        stars = [(v1, v2, v3) for v1 in {x[0] // p, -(-x[0] // p)} for v2 in {x[1] // p, -(-x[1] // p)}
                 for v3 in {x[2] // p, -(-x[2] // p)}
                 if sum(int(x[d] == vd * p) for d, vd in enumerate((v1, v2, v3))) >= 1]
        assert len(stars) == (1, 2, 4)[kind], stars
        want, scale = 0.0, 0.0
        for v in stars:
            sub = _submesh(case, [vd - 1 for vd in v], (2, 2, 2))
            key = (tuple(np.round(np.concatenate(sub.widths), 15)), case.lam)
            if key not in blocks:
                op = condensed.CondensedOperator(sub, case.lam)
                pts, loc = smoother.star_points(sub, (1, 1, 1))
                H = smoother.star_matrix_block(op, (1, 1, 1), pts)
                blocks[key] = (pts, loc, np.linalg.inv(H), smoother.star_weights(sub, (1, 1, 1), loc))
            pts, loc, Hinv, W = blocks[key]
            n1, n2 = sub.N[0], sub.N[1]
            j3, rem = np.divmod(pts, n1 * n2)
            j2, j1 = np.divmod(rem, n1)
            gidx = V.flat((v[0] - 1) * p + j1, (v[1] - 1) * p + j2, (v[2] - 1) * p + j3)
            xs = Hinv @ rg[gidx]
            at = int(np.nonzero(gidx == V.flat(*x))[0][0])
            want += W[at] * xs[at]
            scale = max(scale, np.abs(xs).max())
        errs.append(abs(dug[V.flat(*x)] - want) / scale)
    return max(errs)


@pytest.mark.parametrize("cfg,p", [(2, None), (3, 2), (3, 4), (3, 8), (3, 12), (3, 16), (3, 24), (4, None)])
def test_fullsize_smoother_sampled(cfg, p):
    """The bench-size smoother (every production star kernel: k_star_w at p <= 4 on these meshes,
    k_star_pf, k_star_tm) at sampled vertex, edge and face points against the oracle's dense star
    solves and weights."""
    case = pi.config(cfg, p=p)
    s = _solver(case)
    L = s.nlevels - 1
    rng = np.random.default_rng(7 + cfg + (p or 0))
    n = s.level_info(L)[1]
    rgr = _grid_of(s, L, torch.from_numpy(rng.standard_normal(n)).cuda())
    r = s.new_skel(L)
    s.skel_from_grid(L, torch.from_numpy(rgr).cuda(), r)
    du = s.new_skel(L)
    s.smooth(L, r, du)
    dug = _grid_of(s, L, du)
    err = _sampled_smoother(case, rgr, dug, rng, 6)
    assert err < 1e-11, err
    s.close()


@pytest.mark.parametrize("p,stretch,lam", [(2, None, 0.0), (3, 1.02, 0.4), (4, 1.05, 0.7)])
def test_large_mesh_operators_full_vector(p, stretch, lam):
    """29 x 28 x 28 elements (>= 2960 stars per colour: the warp-per-star kernel k_star_w that the
    p = 2 / 4 levels of configs 3-5 run) -- residual and smoother on every level of the hierarchy
    against the oracle element-wise (full vectors)."""
    from oracle import mg
    k = (29, 28, 28)
    case = pi.small_case(k, p, lam, stretch=stretch)
    s = _solver(case, coarse_rtol=1e-13)
    for l in range(s.nlevels):
        deg = s.level_info(l)[0]
        lv = mg.Level(case.k, case.widths, deg, lam, 7)
        m = lv.mesh
        rng = np.random.default_rng(40 + l)
        u = rng.standard_normal(m.ntot) * m.free_skel
        f = rng.standard_normal(m.ntot) * m.free_skel
        us, fs, r, du = s.new_skel(l), s.new_skel(l), s.new_skel(l), s.new_skel(l)
        s.skel_from_grid(l, torch.from_numpy(u).cuda(), us)
        s.skel_from_grid(l, torch.from_numpy(f).cuda(), fs)
        s.residual(l, us, fs, r)
        s.smooth(l, fs, du)
        rg, dg = _grid_of(s, l, r), _grid_of(s, l, du)
        want_r, want_s = lv.op.residual(u, f), lv.smoother.apply(f)
        for got, want in ((rg, want_r), (dg, want_s)):
            e2 = np.linalg.norm(got - want) / np.linalg.norm(want)
            ei = np.abs(got - want).max() / np.abs(want).max()
            assert e2 < 1e-11 and ei < 1e-10, (l, e2, ei)
    s.close()


@pytest.mark.parametrize("cfg,p,max_cycles", [(2, None, 4), (3, 2, 4), (3, 4, 6), (3, 8, 4), (3, 12, 5), (3, 16, 4),
                                              (3, 24, 5), (3, 32, 4), (1, None, 6)])
def test_fullsize_solve_converges(cfg, p, max_cycles):
    """The bench path at full size: pmg_solve reaches the 1e-10 drop within a handful of cycles
    (P:21); history strictly decreasing."""
    case = pi.config(cfg, p=p)
    s = _solver(case)
    L = s.nlevels - 1
    x = [s.grid_coords(L, d) for d in range(3)]
    f = torch.from_numpy(case.f_nodal(x)).cuda()
    F = s.new_grid()
    s.weak_rhs(f, F)
    u = s.new_grid()
    rep = s.solve(F, u, 1e-10, max_cycles=30)
    assert rep["converged"] and rep["cycles"] <= max_cycles, rep
    h = rep["history"]
    assert all(b < a for a, b in zip(h, h[1:]))
    assert torch.isfinite(u).all()
    s.close()


@pytest.mark.parametrize("n_gpu", [1, 8])
def test_fullsize_config5_converges(n_gpu):
    """BASELINE configs[4] on ONE GPU: the bench's one-GPU slab (64 x 64 x 8, p = 16, 134 M unknowns)
    and the whole 8-GPU problem (64^3, p = 16, 1.07e9 unknowns: the maximum size, ~35 GB of HBM):
    the 1e-10 drop in the paper's handful of cycles, history strictly decreasing, and the final
    residual recomputed from the returned skeleton solution by a separate operator call."""
    case = pi.config(5, n_gpu=n_gpu)
    s = _solver(case)
    L = s.nlevels - 1
    x = [s.grid_coords(L, d) for d in range(3)]
    f = s.new_grid()
    plane = len(x[0]) * len(x[1])
    for z0 in range(0, len(x[2]), 64):             # seeded input generated in z chunks (host memory)
        z1 = min(z0 + 64, len(x[2]))
        f[z0 * plane:z1 * plane] = torch.from_numpy(case.f_nodal([x[0], x[1], x[2][z0:z1]], i3_offset=z0)).cuda()
    F = s.new_grid()
    s.weak_rhs(f, F)
    del f
    u = s.new_grid()
    rep = s.solve(F, u, 1e-10, max_cycles=30)
    assert rep["converged"] and rep["cycles"] <= 4, rep
    h = rep["history"]
    assert all(b < a for a, b in zip(h, h[1:]))
    fh, uh, r = s.new_skel(L), s.new_skel(L), s.new_skel(L)
    s.condense(F, fh)
    s.skel_from_grid(L, u, uh)
    s.residual(L, uh, fh, r)
    rn = s.norm(L, r)
    assert rn <= 1.01e-10 * h[0] and abs(rn - h[-1]) <= 1e-3 * h[-1] + 1e-14 * h[0], (rn, h)
    s.close()


def test_fullsize_config4_manufactured():
    """Config 4: lambda = 100, f = sin x sin y sin z on the stretched 32^3 mesh, p = 16; exact solution
    u = f / 103; the discrete solution is spectrally accurate."""
    case = pi.config(4)
    s = _solver(case)
    L = s.nlevels - 1
    x = [s.grid_coords(L, d) for d in range(3)]
    fn = case.f_nodal(x)
    F = s.new_grid()
    s.weak_rhs(torch.from_numpy(fn).cuda(), F)
    u = s.new_grid()
    rep = s.solve(F, u, 1e-10, max_cycles=40)
    assert rep["converged"], rep
    err = np.abs(u.cpu().numpy() - fn / 103.0).max()
    assert err < 1e-9, err
    s.close()


def test_fullsize_config2_matches_oracle_solve():
    """The bench workload (config 2, 2.1 M unknowns) against a full oracle solve: same cycle count,
    solution within 1e-9 relative."""
    from oracle import condensed, mg
    case = pi.config(2)
    s = _solver(case)
    L = s.nlevels - 1
    x = [s.grid_coords(L, d) for d in range(3)]
    f = case.f_nodal(x)
    F = s.new_grid()
    s.weak_rhs(torch.from_numpy(f).cuda(), F)
    u = s.new_grid()
    rep = s.solve(F, u, 1e-10)
    H = mg.Hierarchy(case.k, case.widths, case.p, case.lam)
    m = H.levels[-1].mesh
    u_o, rep_o = H.solve(condensed.weak_rhs(m, case.f_nodal(m.coords)), 1e-10)
    got = u.cpu().numpy()
    assert rep["cycles"] == rep_o["cycles"]
    assert np.linalg.norm(got - u_o) / np.linalg.norm(u_o) < 1e-9
    s.close()
