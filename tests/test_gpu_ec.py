"""GPU-vs-oracle parity of the element-centred block smoother
through the C ABI: one smoother application per level against oracle/ecsmoother.py (dense LU of
every assembled condensed block) to the north star's 1e-11 per operator application, and whole
solves against the oracle's V-cycle with the same smoother (1e-9 on the solution, identical cycle
counts).  Ragged meshes (k_d not multiples of 3: partial colours), odd and even p, stretched
elements, lambda = 0 and > 0, Neumann faces, boundary blocks."""
import numpy as np
import pytest

import pmg_inputs as pi

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

OP_TOL = 1e-11
SOLVE_TOL = 1e-9

CASES = {
    "k434_p4_lam0.8_stretched": dict(k=(4, 3, 4), p=4, lam=0.8, stretch=1.5, neumann=0),
    "k553_p3_lam0": dict(k=(5, 5, 3), p=3, lam=0.0, stretch=None, neumann=0),
    "k333_p8_lam0": dict(k=(3, 3, 3), p=8, lam=0.0, stretch=None, neumann=0),
    "k422_p5_lam1_neu": dict(k=(4, 2, 2), p=5, lam=1.0, stretch=1.2, neumann=0b100110),
    "k532_p7_lam0": dict(k=(5, 3, 2), p=7, lam=0.0, stretch=1.3, neumann=0),
    "k212_p6_lam2": dict(k=(2, 1, 2), p=6, lam=2.0, stretch=None, neumann=0),
}


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


class Pair:
    def __init__(self, k, p, lam, stretch, neumann, coarse_rtol=1e-13):
        from oracle import mg
        import paper_1808_03595_b200 as pmg
        case = pi.small_case(k, p, lam, stretch=stretch)
        self.case = case
        self.orc = mg.Hierarchy(case.k, case.widths, p, lam, coarse_rtol=coarse_rtol, neumann=neumann,
                                smoother="element")
        self.gpu = pmg.Solver(case.k, case.widths, p, lam, coarse_rtol=coarse_rtol, neumann=neumann, smoother=1)
        self.rng = np.random.default_rng(5)

    def mesh(self, l):
        return self.orc.levels[l].mesh

    def to_skel(self, l, x):
        g = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).cuda()
        s = self.gpu.new_skel(l)
        self.gpu.skel_from_grid(l, g, s)
        return s

    def to_grid(self, l, skel):
        g = self.gpu.new_grid(l)
        self.gpu.skel_to_grid(l, skel, g)
        torch.cuda.synchronize()
        return g.cpu().numpy()

    def rand_skel(self, l):
        m = self.mesh(l)
        return self.rng.standard_normal(m.ntot) * m.free_skel


_PAIRS = {}


def pair(name):
    if name not in _PAIRS:
        _PAIRS[name] = Pair(**CASES[name])
    return _PAIRS[name]


@pytest.mark.parametrize("name", list(CASES))
def test_ec_smooth_parity(name):
    P = pair(name)
    for l in range(1, P.gpu.nlevels):
        sm = P.orc.levels[l].smoother
        u0, r = P.rand_skel(l), P.rand_skel(l)
        u = P.to_skel(l, u0)
        P.gpu.smooth(l, P.to_skel(l, r), u)
        want = sm.apply(r)
        assert rel(P.to_grid(l, u) - u0, want) < OP_TOL, l


@pytest.mark.parametrize("name", list(CASES))
def test_ec_solve_parity(name):
    from oracle import condensed
    P = pair(name)
    m = P.mesh(P.gpu.nlevels - 1)
    F = condensed.weak_rhs(m, pi.uniform_pm1(9, np.arange(m.ntot)))
    u_o, rep_o = P.orc.solve(F, 1e-10)
    ug = P.gpu.new_grid()
    rep = P.gpu.solve(torch.from_numpy(F).cuda(), ug, 1e-10)
    torch.cuda.synchronize()
    assert rep["converged"] and rep["cycles"] == rep_o["cycles"], (rep["cycles"], rep_o["cycles"])
    h, ho = np.array(rep["history"]), np.array(rep_o["history"])
    assert np.all(np.abs(h - ho) <= 1e-8 * ho[0]), (h, ho)
    assert rel(ug.cpu().numpy(), u_o) < SOLVE_TOL


def test_ec_deterministic_and_linear():
    P = pair("k434_p4_lam0.8_stretched")
    l = P.gpu.nlevels - 1
    a, b = P.rand_skel(l), P.rand_skel(l)
    ua, ub, uab, u2 = (P.gpu.new_skel(l) for _ in range(4))
    P.gpu.smooth(l, P.to_skel(l, a), ua)
    P.gpu.smooth(l, P.to_skel(l, b), ub)
    P.gpu.smooth(l, P.to_skel(l, a + 2.0 * b), uab)
    P.gpu.smooth(l, P.to_skel(l, a), u2)
    torch.cuda.synchronize()
    assert torch.equal(ua, u2)
    assert rel(uab.cpu().numpy(), (ua + 2.0 * ub).cpu().numpy()) < 1e-13


def test_ec_converges_faster_than_star_on_gpu():
    """BASELINE configs[0]-like Helmholtz problem at 6^3 elements: the element-centred smoother's
    residual history drops faster per cycle than the star's (more overlap)."""
    import paper_1808_03595_b200 as pmg
    k = (6, 6, 6)
    w = pi.uniform_widths(k, (2 * np.pi,) * 3)
    reps = []
    for sm in (0, 1):
        s = pmg.Solver(k, w, 8, 1.0, smoother=sm)
        f = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, s.level_info(s.nlevels - 1)[2])).cuda()
        F = s.new_grid()
        s.weak_rhs(f, F)
        u = s.new_grid()
        reps.append(s.solve(F, u, 1e-10))
        s.close()
    assert reps[0]["converged"] and reps[1]["converged"]
    assert reps[1]["cycles"] <= reps[0]["cycles"] and reps[1]["rho"] < reps[0]["rho"], (reps[0]["rho"], reps[1]["rho"])


def test_ec_invalid_options():
    import paper_1808_03595_b200 as pmg
    w = [np.ones(2)] * 3
    with pytest.raises(pmg.PmgError):
        pmg.Solver((2, 2, 2), w, 20, 0.0, smoother=1)          # p > 16
    with pytest.raises(pmg.PmgError):
        pmg.Solver((2, 2, 2), w, 4, 0.0, smoother=2)           # unknown smoother
    hub = pmg.Loopback(2)
    with pytest.raises(pmg.PmgError):
        pmg.Solver((2, 2, 4), w[:2] + [np.ones(4)], 4, 0.0, smoother=1, rank=0, nranks=2, loopback=hub)


@pytest.mark.parametrize("p", [4, 8, 13])
def test_ec_kernel_variants_agree(p, monkeypatch):
    """The DMMA kernel (p <= 13, default) and the DFMA kernel (PMG_EC_VARIANT=dfma; the only one
    for p = 14 .. 16) apply the same smoother."""
    import paper_1808_03595_b200 as pmg
    case = pi.small_case((4, 3, 3), p, 0.6, stretch=1.3)
    s = pmg.Solver(case.k, case.widths, p, 0.6, smoother=1)
    l = s.nlevels - 1
    r = torch.from_numpy(np.random.default_rng(p).standard_normal(s.level_info(l)[1])).cuda()
    outs = []
    for var in ("mma", "dfma"):
        monkeypatch.setenv("PMG_EC_VARIANT", var)
        u = s.new_skel(l)
        s.smooth(l, r, u)
        torch.cuda.synchronize()
        outs.append(u.cpu().numpy())
    s.close()
    assert rel(outs[0], outs[1]) < 1e-13


@pytest.mark.parametrize("k,p", [((1, 1, 1), 4), ((1, 2, 3), 3), ((2, 1, 1), 6)])
def test_ec_degenerate_meshes(k, p):
    """One element in some direction: blocks hang over the boundary on both sides (identity padding
    at both block ends) -- smoother and solve still equal the oracle's."""
    from oracle import condensed, mg
    import paper_1808_03595_b200 as pmg
    case = pi.small_case(k, p, 0.9, stretch=None)
    orc = mg.Hierarchy(case.k, case.widths, p, case.lam, coarse_rtol=1e-13, smoother="element")
    m = orc.levels[-1].mesh
    F = condensed.weak_rhs(m, pi.uniform_pm1(9, np.arange(m.ntot)))
    u_o, rep_o = orc.solve(F, 1e-10)
    s = pmg.Solver(case.k, case.widths, p, case.lam, coarse_rtol=1e-13, smoother=1)
    ug = s.new_grid()
    rep = s.solve(torch.from_numpy(F).cuda(), ug, 1e-10)
    torch.cuda.synchronize()
    assert rep["cycles"] == rep_o["cycles"], (rep["cycles"], rep_o["cycles"])
    assert rel(ug.cpu().numpy(), u_o) < SOLVE_TOL
    s.close()


@pytest.mark.parametrize("p", [14, 16])
def test_ec_high_degree_dfma_parity(p):
    """p = 14 .. 16 run the DFMA kernel (the DMMA planes do not fit shared memory): one smoother
    application per level against the oracle's dense-LU blocks on a 2 x 2 x 1 mesh (z faces
    Neumann so that the single element layer has unknowns)."""
    from oracle import mg
    import paper_1808_03595_b200 as pmg
    case = pi.small_case((2, 2, 1), p, 0.8, stretch=1.2)
    orc = mg.Hierarchy(case.k, case.widths, p, 0.8, neumann=0b110000, smoother="element")
    s = pmg.Solver(case.k, case.widths, p, 0.8, neumann=0b110000, smoother=1)
    rng = np.random.default_rng(p)
    for l in range(1, s.nlevels):
        m = orc.levels[l].mesh
        r = rng.standard_normal(m.ntot) * m.free_skel
        rs, us = s.new_skel(l), s.new_skel(l)
        s.skel_from_grid(l, torch.from_numpy(r).cuda(), rs)
        s.smooth(l, rs, us)
        ug = s.new_grid(l)
        s.skel_to_grid(l, us, ug)
        torch.cuda.synchronize()
        assert rel(ug.cpu().numpy(), orc.levels[l].smoother.apply(r)) < OP_TOL, (p, l)
    s.close()
