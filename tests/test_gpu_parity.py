"""GPU-vs-oracle parity through the C ABI (north star: 1e-11 relative per operator application,
1e-9 relative on the final solution), on seeded inputs at sizes the oracle finishes in seconds
that still span several elements/stars per direction and ragged (non-power-of-two, odd p,
stretched) meshes."""
import numpy as np
import pytest

import pmg_inputs as pi

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

OP_TOL = 1e-11
SOLVE_TOL = 1e-9

# Every degree class of the production kernels has a case: p <= 4 (k_star_pf / k_star_w, k_elem_pf),
# 5..8 (k_star_pf, k_elem_pf), 9..16 (k_star_pf<P> with n_S padded to 32, k_elem_pf16), 17..32
# (k_star_tm, k_elem_apply_t); each hierarchy also runs the lower levels' kernels.  p = 32 needs
# ~60 GB of host memory for the oracle's dense p = 32 element Schur complement.
CASES = {
    "k323_p4_lam1.7_stretched": dict(k=(3, 2, 3), p=4, lam=1.7, stretch=1.6),
    "k232_p5_lam0": dict(k=(2, 3, 2), p=5, lam=0.0, stretch=None),
    "k333_p8_lam0": dict(k=(3, 3, 3), p=8, lam=0.0, stretch=None),
    "k422_p3_lam0.5": dict(k=(4, 2, 2), p=3, lam=0.5, stretch=1.3),
    "k332_p2_lam0": dict(k=(3, 3, 2), p=2, lam=0.0, stretch=None),
    "k222_p6_lam2": dict(k=(2, 2, 2), p=6, lam=2.0, stretch=1.2),
    "k222_p12_lam0.3_stretched": dict(k=(2, 2, 2), p=12, lam=0.3, stretch=1.3),
    "k322_p16_lam0": dict(k=(3, 2, 2), p=16, lam=0.0, stretch=None),
    "k223_p13_lam4_stretched": dict(k=(2, 2, 3), p=13, lam=4.0, stretch=1.4),
    "k222_p24_lam1": dict(k=(2, 2, 2), p=24, lam=1.0, stretch=None),
    "k222_p32_lam0": dict(k=(2, 2, 2), p=32, lam=0.0, stretch=None),
}
BIG_HOST = {"k222_p32_lam0": 120}     # GB of available host memory the oracle needs


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def rel_inf(a, b):
    nb = np.abs(b).max() if np.size(b) else 0.0
    return np.abs(a - b).max() / (nb if nb > 0 else 1.0) if np.size(b) else 0.0


def close(a, b, tol):
    """Relative 2-norm error below tol and, alongside (SURVEY 8(c) parity protocol), relative max-norm
    error below 10 tol (a single entry can carry more of the rounding than the 2-norm average)."""
    e2, ei = rel(a, b), rel_inf(a, b)
    return e2 < tol and ei < 10 * tol


class Pair:
    """Oracle hierarchy + GPU solver for the same problem."""

    def __init__(self, k, p, lam, stretch, coarse_rtol=1e-13, schedule=0, neumann=0, periodic=0):
        from oracle import mg
        import paper_1808_03595_b200 as pmg
        case = pi.small_case(k, p, lam, stretch=stretch)
        self.case = case
        self.orc = mg.Hierarchy(case.k, case.widths, p, lam, coarse_rtol=coarse_rtol, schedule=schedule,
                                neumann=neumann, periodic=periodic)
        self.gpu = pmg.Solver(case.k, case.widths, p, lam, coarse_rtol=coarse_rtol, schedule=schedule,
                              neumann=neumann, periodic=periodic)
        assert self.gpu.nlevels == len(self.orc.levels)
        self.rng = np.random.default_rng(11)

    def mesh(self, l):
        return self.orc.levels[l].mesh

    def to_skel(self, l, grid_np):
        g = torch.from_numpy(np.ascontiguousarray(grid_np, dtype=np.float64)).cuda()
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
        need = BIG_HOST.get(name)
        if need:
            import psutil
            if psutil.virtual_memory().available < need * 2 ** 30:
                pytest.skip("oracle needs ~%d GB of host memory for this degree" % need)
        _PAIRS[name] = Pair(**CASES[name])
    return _PAIRS[name]


@pytest.mark.parametrize("name", list(CASES))
def test_coords_and_converters(name):
    P = pair(name)
    for l in range(P.gpu.nlevels):
        m = P.mesh(l)
        for d in range(3):
            assert np.abs(P.gpu.grid_coords(l, d) - m.coords[d]).max() < 1e-14 * max(1.0, m.coords[d].max())
        x = P.rng.standard_normal(m.ntot)
        back = P.to_grid(l, P.to_skel(l, x))
        assert np.array_equal(back, x * m.free_skel)          # exact round trip on free skeleton points
        deg, nskel, ngrid = P.gpu.level_info(l)
        assert deg == m.p and ngrid == m.ntot


@pytest.mark.parametrize("name", list(CASES))
def test_weak_rhs(name):
    from oracle import condensed
    P = pair(name)
    m = P.mesh(P.gpu.nlevels - 1)
    f = P.rng.standard_normal(m.ntot)
    F = P.gpu.new_grid()
    P.gpu.weak_rhs(torch.from_numpy(f).cuda(), F)
    torch.cuda.synchronize()
    assert rel(F.cpu().numpy(), condensed.weak_rhs(m, f)) < 1e-14


@pytest.mark.parametrize("name", list(CASES))
def test_residual_parity(name):
    P = pair(name)
    for l in range(P.gpu.nlevels):
        op = P.orc.levels[l].op
        u, f = P.rand_skel(l), P.rand_skel(l)
        r = P.gpu.new_skel(l)
        P.gpu.residual(l, P.to_skel(l, u), P.to_skel(l, f), r)
        assert close(P.to_grid(l, r), op.residual(u, f), OP_TOL), l
        q = P.gpu.new_skel(l)
        P.gpu.residual(l, P.to_skel(l, u), None, q)              # operator apply
        assert close(P.to_grid(l, q), op.apply(u), OP_TOL), l


@pytest.mark.parametrize("name", list(CASES))
def test_operator_symmetric_on_gpu(name):
    P = pair(name)
    l = P.gpu.nlevels - 1
    a, b = P.to_skel(l, P.rand_skel(l)), P.to_skel(l, P.rand_skel(l))
    Ha, Hb = P.gpu.new_skel(l), P.gpu.new_skel(l)
    P.gpu.residual(l, a, None, Ha)
    P.gpu.residual(l, b, None, Hb)
    x, y = float((Ha * b).sum()), float((a * Hb).sum())
    assert abs(x - y) <= 1e-12 * max(abs(x), 1.0)


@pytest.mark.parametrize("name", list(CASES))
def test_smooth_parity(name):
    P = pair(name)
    for l in range(P.gpu.nlevels):
        sm = P.orc.levels[l].smoother
        u0, r = P.rand_skel(l), P.rand_skel(l)
        u = P.to_skel(l, u0)
        P.gpu.smooth(l, P.to_skel(l, r), u)
        want = u0 + sm.apply(r)
        assert close(P.to_grid(l, u) - u0, want - u0, OP_TOL), l


@pytest.mark.parametrize("name", [n for n in CASES if CASES[n]["p"] > 2])
def test_transfer_parity(name):
    P = pair(name)
    for l in range(1, P.gpu.nlevels):
        T = P.orc.transfers[l]
        rf = P.rand_skel(l)
        fc = P.gpu.new_skel(l - 1)
        P.gpu.restrict(l, P.to_skel(l, rf), fc)
        assert close(P.to_grid(l - 1, fc), T.restrict(rf), OP_TOL), l
        uc, uf0 = P.rand_skel(l - 1), P.rand_skel(l)
        uf = P.to_skel(l, uf0)
        P.gpu.prolong(l, P.to_skel(l - 1, uc), uf)
        assert close(P.to_grid(l, uf) - uf0, T.prolong(uc), OP_TOL), l


@pytest.mark.parametrize("name", list(CASES))
def test_condense_recover_parity(name):
    P = pair(name)
    L = P.gpu.nlevels - 1
    m = P.mesh(L)
    op = P.orc.levels[L].op
    F = P.rng.standard_normal(m.ntot) * m.free
    Fd = torch.from_numpy(F).cuda()
    fh = P.gpu.new_skel(L)
    P.gpu.condense(Fd, fh)
    assert close(P.to_grid(L, fh), op.condense(F), OP_TOL)
    uh = P.rand_skel(L)
    ug = P.gpu.new_grid()
    P.gpu.recover(P.to_skel(L, uh), Fd, ug)
    torch.cuda.synchronize()
    assert close(ug.cpu().numpy(), op.recover(uh, F), OP_TOL)


@pytest.mark.parametrize("name", list(CASES))
def test_vcycle_parity(name):
    P = pair(name)
    L = P.gpu.nlevels - 1
    u0, f = P.rand_skel(L), P.rand_skel(L)
    u = P.to_skel(L, u0)
    P.gpu.vcycle(u, P.to_skel(L, f))
    want = P.orc.vcycle(u0, f)
    assert close(P.to_grid(L, u), want, OP_TOL)


@pytest.mark.parametrize("name", list(CASES))
def test_solve_parity(name):
    from oracle import condensed
    P = pair(name)
    L = P.gpu.nlevels - 1
    m = P.mesh(L)
    f = pi.uniform_pm1(5, np.arange(m.ntot))
    F = condensed.weak_rhs(m, f)
    u_orc, rep_o = P.orc.solve(F, 1e-10)
    ug = P.gpu.new_grid()
    rep = P.gpu.solve(torch.from_numpy(F).cuda(), ug, 1e-10)
    torch.cuda.synchronize()
    assert rep["converged"] and rep["cycles"] == rep_o["cycles"]
    assert close(ug.cpu().numpy(), u_orc, SOLVE_TOL)
    assert abs(rep["r0"] - rep_o["r0"]) <= 1e-12 * rep_o["r0"]
    # phase times of the report: all measured, the coarse solves inside the cycle loop
    assert rep["t_condense"] > 0 and rep["t_cycles"] > 0 and rep["t_recover"] > 0
    assert 0 < rep["t_coarse"] <= rep["t_cycles"]


def test_smoother_deterministic():
    P = pair("k333_p8_lam0")
    l = P.gpu.nlevels - 1
    r = P.to_skel(l, P.rand_skel(l))
    u1, u2 = P.gpu.new_skel(l), P.gpu.new_skel(l)
    P.gpu.smooth(l, r, u1)
    P.gpu.smooth(l, r, u2)
    torch.cuda.synchronize()
    assert torch.equal(u1, u2)


def test_invalid_arguments_fail_loudly():
    import paper_1808_03595_b200 as pmg
    with pytest.raises(pmg.PmgError):
        pmg.Solver((2, 2, 2), [np.ones(2)] * 3, 1, 0.0)           # p < 2
    with pytest.raises(pmg.PmgError):
        pmg.Solver((2, 2, 2), [np.array([1.0, -1.0])] * 3, 4, 0.0)  # negative width
    with pytest.raises(pmg.PmgError):
        pmg.Solver((2, 2, 2), [np.ones(2)] * 3, 4, -1.0)          # lambda < 0
    P = pair("k232_p5_lam0")
    with pytest.raises(pmg.PmgError):
        P.gpu.restrict(0, P.gpu.new_skel(0), P.gpu.new_skel(0))   # no level below 0


@pytest.mark.parametrize("name", ["k333_p8_lam0", "k422_p3_lam0.5", "k332_p2_lam0"])
def test_coarse_cg_paths_agree(name, monkeypatch):
    """The persistent cooperative coarse CG (stencil + rank-one element corrections) and the
    multi-kernel CG (element operator) are two evaluations of the same Jacobi-PCG iteration."""
    import paper_1808_03595_b200 as pmg
    P = pair(name)
    case = P.case
    L = P.gpu.nlevels - 1
    f = P.rand_skel(L)
    outs = []
    for env in ("0", "1"):
        monkeypatch.setenv("PMG_COARSE_MULTIKERNEL", env)
        s = pmg.Solver(case.k, case.widths, case.p, case.lam, coarse_rtol=1e-13)
        u = s.new_skel(L)
        fs = torch.from_numpy(np.ascontiguousarray(f)).cuda()
        fh = s.new_skel(L)
        s.skel_from_grid(L, fs, fh)
        s.vcycle(u, fh)
        g = s.new_grid(L)
        s.skel_to_grid(L, u, g)
        torch.cuda.synchronize()
        outs.append(g.cpu().numpy())
        s.close()
    assert rel(outs[0], outs[1]) < 1e-11
    assert close(outs[0], P.orc.vcycle(np.zeros_like(f), f), OP_TOL)


@pytest.mark.parametrize("kind", ["registers", "ell"])
@pytest.mark.parametrize("name", ["k323_p4_lam1.7_stretched", "k333_p8_lam0", "k332_p2_lam0"])
def test_pipelined_coarse_cg_matches_standard(name, kind, monkeypatch):
    """The single-barrier (pipelined) coarse CG used at the performance tolerance -- register-
    resident (one thread per unknown) or grid-stride over ELL rows (large coarse systems) --
    reproduces the standard two-barrier Jacobi-PCG: same coarse iteration count over a solve (+-1
    per coarse solve), and V-cycle outputs that agree to the coarse tolerance's accuracy; against
    the oracle's standard PCG V-cycle at the same tolerance likewise."""
    import paper_1808_03595_b200 as pmg
    from oracle import mg
    P = pair(name)
    case = P.case
    L = P.gpu.nlevels - 1
    f = P.rand_skel(L)
    outs, its = [], []
    envs = [("1", "0"), ("0", "0")] if kind == "registers" else [("0", "1"), ("0", "0")]
    for gv, ell in envs:
        monkeypatch.setenv("PMG_COARSE_GV", gv)
        monkeypatch.setenv("PMG_COARSE_ELL", ell)
        s = pmg.Solver(case.k, case.widths, case.p, case.lam, coarse_rtol=1e-10)
        u = s.new_skel(L)
        fs = torch.from_numpy(np.ascontiguousarray(f)).cuda()
        fh = s.new_skel(L)
        s.skel_from_grid(L, fs, fh)
        s.vcycle(u, fh)
        g = s.new_grid(L)
        s.skel_to_grid(L, u, g)
        F = torch.from_numpy(np.ascontiguousarray(np.random.default_rng(21).standard_normal(g.numel()))).cuda()
        Fw = s.new_grid(L)
        s.weak_rhs(F, Fw)
        ug = s.new_grid(L)
        rep = s.solve(Fw, ug, 1e-10)
        torch.cuda.synchronize()
        outs.append(g.cpu().numpy())
        its.append((rep["coarse_iters"], rep["cycles"]))
        s.close()
    assert rel(outs[0], outs[1]) < 1e-7
    # the pipelined recurrence's recursive residual may cross the threshold an iteration or two
    # earlier than the standard one (residual gap near rtol = 1e-10): +-2 per coarse solve
    assert its[0][1] == its[1][1] and abs(its[0][0] - its[1][0]) <= 2 * its[0][1], its
    orc = mg.Hierarchy(case.k, case.widths, case.p, case.lam, coarse_rtol=1e-10)
    assert rel(outs[0], orc.vcycle(np.zeros_like(f), f)) < 1e-7


@pytest.mark.parametrize("schedule", [0, 1])
@pytest.mark.parametrize("name", ["k323_p4_lam1.7_stretched", "k232_p5_lam0", "k333_p8_lam0", "k332_p2_lam0"])
def test_krylov_solve_parity(name, schedule):
    """Alg. 5 (ipCG + V-cycle preconditioner; kMG / kvMG) on the GPU against the oracle's verbatim
    Alg. 5: same iteration count and residual history, solution within the solve tolerance."""
    import paper_1808_03595_b200 as pmg
    from oracle import condensed, mg
    cfg = CASES[name]
    case = pi.small_case(cfg["k"], cfg["p"], cfg["lam"], stretch=cfg["stretch"])
    orc = mg.Hierarchy(case.k, case.widths, case.p, case.lam, coarse_rtol=1e-13, schedule=schedule)
    m = orc.levels[-1].mesh
    F = condensed.weak_rhs(m, pi.uniform_pm1(6, np.arange(m.ntot)))
    u_o, rep_o = orc.solve_ipcg(F, 1e-10)
    s = pmg.Solver(case.k, case.widths, case.p, case.lam, coarse_rtol=1e-13, schedule=schedule, solver=1)
    ug = s.new_grid()
    rep = s.solve(torch.from_numpy(F).cuda(), ug, 1e-10)
    torch.cuda.synchronize()
    assert rep["converged"] and rep["cycles"] == rep_o["cycles"], (rep["cycles"], rep_o["cycles"])
    h, ho = np.array(rep["history"]), np.array(rep_o["history"])
    assert np.all(np.abs(h - ho) <= 1e-8 * ho[0]), (h, ho)
    assert close(ug.cpu().numpy(), u_o, SOLVE_TOL)
    s.close()


TABLE_SOLVERS = {"MG": dict(solver=0, schedule=0), "kMG": dict(solver=1, schedule=0), "kvMG": dict(solver=1, schedule=1)}


def _gpu_iters(k, widths, p, solver):
    import paper_1808_03595_b200 as pmg
    s = pmg.Solver(k, widths, p, 0.0, **TABLE_SOLVERS[solver])
    f = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, s.level_info(s.nlevels - 1)[2])).cuda()
    F = s.new_grid()
    s.weak_rhs(f, F)
    u = s.new_grid()
    rep = s.solve(F, u, 1e-10, max_cycles=200)
    torch.cuda.synchronize()
    s.close()
    return rep


@pytest.mark.parametrize("p", [4, 8, 16, 32])
@pytest.mark.parametrize("alpha", [1, 1.5, 2])
def test_gpu_iteration_counts_match_paper_table(alpha, p):
    """All 36 cells of Table tab:stretched_poly_iterations -- MG, kMG and kvMG (Alg. 4 / 5,
    nu = 1 or 2^(L-l)) at p = 4, 8, 16, 32 and expansion factor alpha = 1, 1.5, 2 (reading R13) -- on
    the GPU path: 8^3 elements on (0, 2 pi)^3, lambda = 0, random RHS, 1e-10 drop; within +-1 of the
    printed count (the paper's random RHS and coarse tolerance are unstated)."""
    import json
    import math
    import os
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "stretched_poly_iterations.json")))
    w = [pi.geometric_widths(8, 2 * math.pi, alpha)] * 3
    for solver in ("MG", "kMG", "kvMG"):
        want = gold[solver][str(alpha)][gold["p"].index(p)]
        rep = _gpu_iters((8, 8, 8), w, p, solver)
        assert rep["converged"] and abs(rep["cycles"] - want) <= 1, (solver, rep["cycles"], want)


def test_gpu_anisotropic_meshes_paper_claims():
    """Sec. 5.3: 8^3 elements of degree 16 on (0, 2 pi AR) x (0, pi ceil(AR/2)) x (0, 2 pi).
    The figure's data are not in the source, so the text's claims are checked: MG needs about three
    iterations at AR = 1 and "increases from three to sixty" at AR = 48; Krylov acceleration "helps,
    but does not completely remove the effect"; more smoothing per level (kvMG) "keeps the number of
    iterations mostly stable until AR = 8"."""
    import math

    def iters(AR, solver):
        L = (2 * math.pi * AR, math.pi * math.ceil(AR / 2), 2 * math.pi)
        return _gpu_iters((8, 8, 8), pi.uniform_widths((8, 8, 8), L), 16, solver)["cycles"]
    mg1, mg48 = iters(1, "MG"), iters(48, "MG")
    k1, k48 = iters(1, "kMG"), iters(48, "kMG")
    kv1, kv8 = iters(1, "kvMG"), iters(8, "kvMG")
    assert 2 <= mg1 <= 4 and 40 <= mg48 <= 80, (mg1, mg48)
    assert k48 < mg48 / 2 and k48 > 2 * k1, (k1, k48, mg48)
    assert kv8 <= kv1 + 2, (kv1, kv8)


@pytest.mark.parametrize("k,p", [((1, 1, 1), 4), ((1, 2, 3), 3), ((1, 1, 4), 2), ((2, 1, 1), 6)])
def test_degenerate_meshes(k, p):
    """Edge cases: one element per direction (k = 1: every element face is Dirichlet, the condensed
    system is empty or one-dimensional per line) -- the solve must still equal the oracle's."""
    import paper_1808_03595_b200 as pmg
    from oracle import condensed, mg
    case = pi.small_case(k, p, 0.9, stretch=None)
    orc = mg.Hierarchy(case.k, case.widths, p, case.lam, coarse_rtol=1e-13)
    m = orc.levels[-1].mesh
    F = condensed.weak_rhs(m, pi.uniform_pm1(9, np.arange(m.ntot)))
    u_o, rep_o = orc.solve(F, 1e-10)
    s = pmg.Solver(case.k, case.widths, p, case.lam, coarse_rtol=1e-13)
    ug = s.new_grid()
    rep = s.solve(torch.from_numpy(F).cuda(), ug, 1e-10)
    torch.cuda.synchronize()
    assert rep["cycles"] == rep_o["cycles"], (rep["cycles"], rep_o["cycles"])
    assert close(ug.cpu().numpy(), u_o, SOLVE_TOL)
    s.close()


def test_solve_host_and_report_paths():
    """pmg_solve_host (host buffers, pageable and pinned) equals the device solve bitwise; repeated
    solves are bitwise deterministic (graph replay); max_cycles too small returns PMG_ENOCONV with
    the report filled and u written."""
    import paper_1808_03595_b200 as pmg
    from oracle import condensed
    P = pair("k323_p4_lam1.7_stretched")
    s = P.gpu
    L = s.nlevels - 1
    m = P.mesh(L)
    F = condensed.weak_rhs(m, pi.uniform_pm1(12, np.arange(m.ntot)))
    Fd = torch.from_numpy(F).cuda()
    u1, u2 = s.new_grid(), s.new_grid()
    r1 = s.solve(Fd, u1, 1e-10)
    r2 = s.solve(Fd, u2, 1e-10)
    torch.cuda.synchronize()
    assert torch.equal(u1, u2) and r1["history"] == r2["history"]
    uh = np.zeros_like(F)
    rh = s.solve_host(np.ascontiguousarray(F), uh, 1e-10)
    assert rh["cycles"] == r1["cycles"] and np.array_equal(uh, u1.cpu().numpy())
    Fp = torch.from_numpy(F).pin_memory()
    up = torch.zeros_like(Fp).pin_memory()
    s.solve_host(Fp, up, 1e-10)
    assert np.array_equal(up.numpy(), uh)
    u3 = s.new_grid()
    r3 = s.solve(Fd, u3, 1e-10, max_cycles=1)
    torch.cuda.synchronize()
    assert r3["status"] == pmg.PMG_ENOCONV and not r3["converged"] and r3["cycles"] == 1
    assert r3["r_final"] < r3["r0"] and float(u3.abs().max()) > 0


NEUMANN_CASES = {
    "k323_p4_neu_x": dict(k=(3, 2, 3), p=4, lam=1.7, stretch=1.6, neumann=0b000011),
    "k232_p5_neu_mixed": dict(k=(2, 3, 2), p=5, lam=0.0, stretch=None, neumann=0b100110),
    "k333_p8_neu_all": dict(k=(3, 3, 3), p=8, lam=0.9, stretch=None, neumann=0b111111),
    "k332_p2_neu_z": dict(k=(3, 3, 2), p=2, lam=0.0, stretch=None, neumann=0b110000),
}
_NPAIRS = {}


def npair(name):
    if name not in _NPAIRS:
        _NPAIRS[name] = Pair(**NEUMANN_CASES[name])
    return _NPAIRS[name]


@pytest.mark.parametrize("name", list(NEUMANN_CASES))
def test_neumann_operators_parity(name):
    """Homogeneous Neumann faces (NEXT-3): residual, smoother, restriction,
    prolongation and V-cycle against the oracle on the same inputs, per-operator tolerance."""
    P = npair(name)
    L = P.gpu.nlevels - 1
    for l in range(L + 1):
        orc = P.orc.levels[l]
        u = P.rand_skel(l)
        f = P.rand_skel(l)
        r = P.gpu.new_skel(l)
        P.gpu.residual(l, P.to_skel(l, u), P.to_skel(l, f), r)
        assert close(P.to_grid(l, r), orc.op.residual(u, f), OP_TOL)
        du = P.gpu.new_skel(l)
        P.gpu.smooth(l, P.to_skel(l, f), du)
        assert close(P.to_grid(l, du), orc.smoother.apply(f), OP_TOL)
        if l >= 1:
            T = P.orc.transfers[l]
            fc = P.gpu.new_skel(l - 1)
            P.gpu.restrict(l, P.to_skel(l, f), fc)
            assert close(P.to_grid(l - 1, fc), T.restrict(f), OP_TOL)
            uc = P.rand_skel(l - 1)
            uf = P.gpu.new_skel(l)
            P.gpu.prolong(l, P.to_skel(l - 1, uc), uf)
            assert close(P.to_grid(l, uf), T.prolong(uc), OP_TOL)
    f = P.rand_skel(L)
    u = P.gpu.new_skel(L)
    P.gpu.vcycle(u, P.to_skel(L, f))
    assert close(P.to_grid(L, u), P.orc.vcycle(np.zeros_like(f), f), OP_TOL)


@pytest.mark.parametrize("name", list(NEUMANN_CASES))
def test_neumann_solve_parity(name):
    from oracle import condensed
    P = npair(name)
    L = P.gpu.nlevels - 1
    m = P.mesh(L)
    F = condensed.weak_rhs(m, pi.uniform_pm1(5, np.arange(m.ntot)))
    u_orc, rep_o = P.orc.solve(F, 1e-10)
    ug = P.gpu.new_grid()
    rep = P.gpu.solve(torch.from_numpy(F).cuda(), ug, 1e-10)
    torch.cuda.synchronize()
    assert rep["converged"] and rep["cycles"] == rep_o["cycles"], (rep["cycles"], rep_o["cycles"])
    assert close(ug.cpu().numpy(), u_orc, SOLVE_TOL)


@pytest.mark.parametrize("neu,kind", [(0b111111, "cos"), (0b111100, "sin")])
def test_neumann_manufactured_on_gpu(neu, kind):
    """lambda = 1 on (0, pi)^3, 4^3 elements, p = 8: u = cos x cos y cos z (all faces Neumann) or
    sin x cos y cos z (Dirichlet x faces); f = 4 u; the GPU solve reproduces u to spectral accuracy."""
    import math
    import paper_1808_03595_b200 as pmg
    k = (4, 4, 4)
    s = pmg.Solver(k, pi.uniform_widths(k, (math.pi,) * 3), 8, 1.0, neumann=neu)
    L = s.nlevels - 1
    x = [s.grid_coords(L, d) for d in range(3)]
    X3, X2, X1 = np.meshgrid(x[2], x[1], x[0], indexing="ij")
    ue = ((np.cos(X1) if kind == "cos" else np.sin(X1)) * np.cos(X2) * np.cos(X3)).ravel()
    F = s.new_grid()
    s.weak_rhs(torch.from_numpy(4.0 * ue).cuda(), F)
    u = s.new_grid()
    rep = s.solve(F, u, 1e-12)
    torch.cuda.synchronize()
    assert rep["converged"]
    assert np.abs(u.cpu().numpy() - ue).max() < 1e-6
    s.close()


def test_neumann_invalid_options():
    import paper_1808_03595_b200 as pmg
    case = pi.small_case((2, 2, 2), 4, 0.0)
    with pytest.raises(pmg.PmgError):
        pmg.Solver(case.k, case.widths, 4, 0.0, neumann=63)      # singular all-Neumann Poisson
    with pytest.raises(pmg.PmgError):
        pmg.Solver(case.k, case.widths, 4, 1.0, neumann=64)


HMG_CASES = {   # coarse levels above the 1500-unknown dense limit: at least two h-levels
    "k888_p4_lam0.6": dict(k=(8, 8, 8), p=4, lam=0.6, stretch=1.3, neumann=0),
    "k1688_p2_lam0": dict(k=(16, 8, 8), p=2, lam=0.0, stretch=None, neumann=0),        # L = 0: CG only
    "k884_p4_neu": dict(k=(8, 8, 4), p=4, lam=0.9, stretch=None, neumann=0b110011),
    # four h-levels (16x16x8 -> 8x8x4 -> 4x4x2 -> 2x2x2, semi-coarsening in x3), stretched widths
    "k16168_p2_stretch": dict(k=(16, 16, 8), p=2, lam=0.3, stretch=1.2, neumann=0),
    "k16816_p2_neu": dict(k=(16, 8, 16), p=2, lam=0.0, stretch=1.1, neumann=0b000011),
}


@pytest.mark.parametrize("name", list(HMG_CASES))
def test_hmg_coarse_solver_parity(name):
    """The h-multigrid preconditioned coarse CG (NEXT-2, reading R16) forced on small meshes: the
    V-cycle and the solve against the oracle running the same preconditioner (oracle/hmg.py)."""
    import paper_1808_03595_b200 as pmg
    from oracle import condensed, mg
    cfg = HMG_CASES[name]
    case = pi.small_case(cfg["k"], cfg["p"], cfg["lam"], stretch=cfg["stretch"])
    orc = mg.Hierarchy(case.k, case.widths, case.p, case.lam, coarse_rtol=1e-13, neumann=cfg["neumann"],
                       coarse_solver="hmg")
    s = pmg.Solver(case.k, case.widths, case.p, case.lam, coarse_rtol=1e-13, neumann=cfg["neumann"],
                   coarse_solver=2)
    L = s.nlevels - 1
    m = orc.levels[-1].mesh
    f = np.random.default_rng(3).standard_normal(m.ntot) * m.free_skel
    fs = s.new_skel(L)
    s.skel_from_grid(L, torch.from_numpy(f).cuda(), fs)
    u = s.new_skel(L)
    s.vcycle(u, fs)
    g = s.new_grid(L)
    s.skel_to_grid(L, u, g)
    torch.cuda.synchronize()
    assert close(g.cpu().numpy(), orc.vcycle(np.zeros_like(f), f), OP_TOL)
    F = condensed.weak_rhs(m, pi.uniform_pm1(8, np.arange(m.ntot)))
    u_o, rep_o = orc.solve(F, 1e-10)
    ug = s.new_grid()
    rep = s.solve(torch.from_numpy(F).cuda(), ug, 1e-10)
    torch.cuda.synchronize()
    assert rep["cycles"] == rep_o["cycles"] and close(ug.cpu().numpy(), u_o, SOLVE_TOL)
    s.close()


def test_hmg_recurrence_true_residual():
    """The h-multigrid CG updates q = H z + beta q by recurrence (one operator application per
    iteration), so its recursive residual can drift from f - H x.  On a 32 x 32 x 16-element p = 2
    mesh (L = 0: the V-cycle is the coarse CG alone, four h-levels) solved to 1e-12, the TRUE residual
    recomputed by the residual kernel must still be below 1e-10 of ||f||."""
    import paper_1808_03595_b200 as pmg
    k = (32, 32, 16)
    case = pi.small_case(k, 2, 0.0, stretch=1.1)
    s = pmg.Solver(case.k, case.widths, 2, 0.0, coarse_rtol=1e-12, coarse_solver=2)
    L = s.nlevels - 1
    assert L == 0
    n = s.level_info(0)[2]
    g = s.new_grid(0)
    g.copy_(torch.from_numpy(np.random.default_rng(5).standard_normal(n)))
    f = s.new_skel(0)
    s.skel_from_grid(0, g, f)
    u = s.new_skel(0)
    s.vcycle(u, f)
    r = s.new_skel(0)
    s.residual(0, u, f, r)
    torch.cuda.synchronize()
    assert torch.linalg.norm(r).item() <= 1e-10 * torch.linalg.norm(f).item()
    s.close()


def test_hmg_auto_on_large_mesh_matches_jacobi():
    """32^3 elements at p = 4 (coarse 32^3 at p0 = 2, 226 k unknowns): the automatic choice takes the
    h-multigrid coarse CG; the solve agrees with the Jacobi-PCG one and needs far fewer coarse
    iterations."""
    import paper_1808_03595_b200 as pmg
    k = (32, 32, 32)
    w = pi.uniform_widths(k, (1.0,) * 3)
    outs = []
    for cs in (0, 1):
        s = pmg.Solver(k, w, 4, 0.0, coarse_solver=cs)
        f = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, s.level_info(s.nlevels - 1)[2])).cuda()
        F = s.new_grid()
        s.weak_rhs(f, F)
        u = s.new_grid()
        rep = s.solve(F, u, 1e-10)
        torch.cuda.synchronize()
        outs.append((u.cpu().numpy(), rep))
        s.close()
    (u0, r0), (u1, r1) = outs
    assert r0["converged"] and r1["converged"] and r0["cycles"] == r1["cycles"]
    assert np.linalg.norm(u0 - u1) <= 1e-8 * np.linalg.norm(u1)
    assert r0["coarse_iters"] * 5 < r1["coarse_iters"], (r0["coarse_iters"], r1["coarse_iters"])


@pytest.mark.parametrize("solver", [0, 1])
def test_zero_rhs_returns_zero(solver):
    """Degenerate input: F = 0 gives r0 = 0, no cycle, u = 0 (as the oracle's Alg. 4 loop)."""
    import paper_1808_03595_b200 as pmg
    from oracle import mg
    case = pi.small_case((3, 2, 2), 4, 0.5, stretch=1.2)
    s = pmg.Solver(case.k, case.widths, 4, 0.5, solver=solver)
    F = s.new_grid()
    u = s.new_grid()
    u.fill_(7.0)
    rep = s.solve(F, u, 1e-10)
    torch.cuda.synchronize()
    orc = mg.Hierarchy(case.k, case.widths, 4, 0.5)
    u_o, rep_o = orc.solve(np.zeros(F.numel()), 1e-10)
    assert rep["converged"] and rep["cycles"] == rep_o["cycles"] == 0 and rep["r0"] == 0.0
    assert float(u.abs().max()) == 0.0 and np.abs(u_o).max() == 0.0
    s.close()


@pytest.mark.parametrize("name", ["k323_p4_lam1.7_stretched", "k422_p3_lam0.5", "k332_p2_lam0"])
def test_warp_star_kernel_forced_parity(name, monkeypatch):
    """The warp-per-star smoother kernel (k_star_w, p <= 4) that the large meshes of configs 3-5 run on
    their p = 2 / 4 levels, forced onto the ragged parity meshes (every star boundary case: padded
    lines, Dirichlet corners, stretched widths) and compared with the oracle on every level."""
    import paper_1808_03595_b200 as pmg
    monkeypatch.setenv("PMG_STAR_W_MIN", "0")
    P = pair(name)
    case = P.case
    s = pmg.Solver(case.k, case.widths, case.p, case.lam, coarse_rtol=1e-13)
    for l in range(s.nlevels):
        sm = P.orc.levels[l].smoother
        r = P.rand_skel(l)
        rs = s.new_skel(l)
        s.skel_from_grid(l, torch.from_numpy(r).cuda(), rs)
        du = s.new_skel(l)
        s.smooth(l, rs, du)
        g = s.new_grid(l)
        s.skel_to_grid(l, du, g)
        torch.cuda.synchronize()
        assert close(g.cpu().numpy(), sm.apply(r), OP_TOL), l
    s.close()


# periodic directions: every kernel family (k_star_pf / k_star_w at
# p <= 4, k_star16 at 5..16, k_star_tm above; k_elem_pf, k_elem16, k_elem_apply_t; transfers;
# condensation / recovery) on wrapped meshes
PERIODIC_CASES = {
    "k423_p4_per_x": dict(k=(4, 2, 3), p=4, lam=0.3, stretch=1.3, periodic=0b001),
    "k324_p8_per_yz": dict(k=(3, 2, 4), p=8, lam=0.0, stretch=None, periodic=0b110),
    "k224_p16_per_xyz": dict(k=(2, 2, 4), p=16, lam=1.1, stretch=None, periodic=0b111),
    "k422_p12_per_x_neu_z": dict(k=(4, 2, 2), p=12, lam=0.5, stretch=1.2, periodic=0b001, neumann=0b110000),
    "k243_p3_per_y": dict(k=(2, 4, 3), p=3, lam=0.0, stretch=None, periodic=0b010),
    "k222_p20_per_x": dict(k=(2, 2, 2), p=20, lam=0.7, stretch=None, periodic=0b001),
}
_PPAIRS = {}


def ppair(name):
    if name not in _PPAIRS:
        _PPAIRS[name] = Pair(**PERIODIC_CASES[name])
    return _PPAIRS[name]


@pytest.mark.parametrize("name", list(PERIODIC_CASES))
def test_periodic_operators_parity(name):
    """Residual, smoother, restriction, prolongation on every level, condensation / recovery and the
    V-cycle against the oracle's wrapped operators (per-operator tolerance)."""
    P = ppair(name)
    L = P.gpu.nlevels - 1
    for l in range(L + 1):
        orc = P.orc.levels[l]
        u, f = P.rand_skel(l), P.rand_skel(l)
        r = P.gpu.new_skel(l)
        P.gpu.residual(l, P.to_skel(l, u), P.to_skel(l, f), r)
        assert close(P.to_grid(l, r), orc.mesh.fill_periodic(orc.op.residual(u, f)), OP_TOL), l
        du = P.gpu.new_skel(l)
        P.gpu.smooth(l, P.to_skel(l, f), du)
        assert close(P.to_grid(l, du), orc.mesh.fill_periodic(orc.smoother.apply(f)), OP_TOL), l
        if l >= 1:
            T = P.orc.transfers[l]
            fc = P.gpu.new_skel(l - 1)
            P.gpu.restrict(l, P.to_skel(l, f), fc)
            assert close(P.to_grid(l - 1, fc), P.orc.levels[l - 1].mesh.fill_periodic(T.restrict(f)), OP_TOL), l
            uc = P.rand_skel(l - 1)
            uf = P.gpu.new_skel(l)
            P.gpu.prolong(l, P.to_skel(l - 1, uc), uf)
            assert close(P.to_grid(l, uf), orc.mesh.fill_periodic(T.prolong(uc)), OP_TOL), l
    m = P.mesh(L)
    op = P.orc.levels[L].op
    F = P.rng.standard_normal(m.ntot) * m.free
    Fd = torch.from_numpy(F).cuda()
    fh = P.gpu.new_skel(L)
    P.gpu.condense(Fd, fh)
    assert close(P.to_grid(L, fh), m.fill_periodic(op.condense(F)), OP_TOL)
    uh = P.rand_skel(L)
    ug = P.gpu.new_grid()
    P.gpu.recover(P.to_skel(L, uh), Fd, ug)
    torch.cuda.synchronize()
    assert close(ug.cpu().numpy(), m.fill_periodic(op.recover(uh, F)), OP_TOL)
    f = P.rand_skel(L)
    u = P.gpu.new_skel(L)
    P.gpu.vcycle(u, P.to_skel(L, f))
    assert close(P.to_grid(L, u), m.fill_periodic(P.orc.vcycle(np.zeros_like(f), f)), OP_TOL)


@pytest.mark.parametrize("name", list(PERIODIC_CASES))
def test_periodic_solve_parity(name):
    from oracle import condensed
    P = ppair(name)
    L = P.gpu.nlevels - 1
    m = P.mesh(L)
    F = condensed.weak_rhs(m, pi.uniform_pm1(5, np.arange(m.ntot)))
    u_orc, rep_o = P.orc.solve(F, 1e-10)
    ug = P.gpu.new_grid()
    rep = P.gpu.solve(torch.from_numpy(F).cuda(), ug, 1e-10)
    torch.cuda.synchronize()
    assert rep["converged"] and rep["cycles"] == rep_o["cycles"], (rep["cycles"], rep_o["cycles"])
    assert close(ug.cpu().numpy(), u_orc, SOLVE_TOL)


@pytest.mark.parametrize("per", [0b001, 0b111])
def test_periodic_manufactured_on_gpu(per):
    """lambda = 1, f = 4 u: u = cos x cos y cos z fully periodic on (0, 2 pi)^3, or u = cos x sin y sin z
    periodic in x with Dirichlet y, z faces on (0, 2 pi) x (0, pi)^2; 4 x 2 x 2 elements, p = 8: the
    GPU solve reproduces u to spectral accuracy, duplicate planes included."""
    import math
    import paper_1808_03595_b200 as pmg
    k = (4, 2, 2)
    Lb = (2 * math.pi,) * 3 if per == 0b111 else (2 * math.pi, math.pi, math.pi)
    s = pmg.Solver(k, pi.uniform_widths(k, Lb), 8, 1.0, periodic=per)
    L = s.nlevels - 1
    x = [s.grid_coords(L, d) for d in range(3)]
    X3, X2, X1 = np.meshgrid(x[2], x[1], x[0], indexing="ij")
    ue = (np.cos(X1) * ((np.cos(X2) * np.cos(X3)) if per == 0b111 else (np.sin(X2) * np.sin(X3)))).ravel()
    F = s.new_grid()
    s.weak_rhs(torch.from_numpy(4.0 * ue).cuda(), F)
    u = s.new_grid()
    rep = s.solve(F, u, 1e-12)
    torch.cuda.synchronize()
    assert rep["converged"]
    assert np.abs(u.cpu().numpy() - ue).max() < 1e-5
    s.close()


def test_periodic_translation_invariance_on_gpu():
    """Uniform elements, periodic in x: the GPU solution of the right-hand side shifted by one element
    along x is the shifted solution."""
    import paper_1808_03595_b200 as pmg
    k, p = (6, 2, 3), 8
    s = pmg.Solver(k, pi.uniform_widths(k, (1.0, 0.7, 0.9)), p, 0.3, periodic=0b001, coarse_rtol=1e-13)
    N = (k[0] * p + 1, k[1] * p + 1, k[2] * p + 1)
    g = np.random.default_rng(5).uniform(-1, 1, (N[2], N[1], N[0] - 1))

    def solve(gg):
        f = np.concatenate([gg, gg[:, :, :1]], axis=2).ravel()
        F = s.new_grid()
        s.weak_rhs(torch.from_numpy(f).cuda(), F)
        u = s.new_grid()
        rep = s.solve(F, u, 1e-12)
        torch.cuda.synchronize()
        return u.cpu().numpy().reshape(N[2], N[1], N[0])[:, :, :N[0] - 1], rep
    u1, r1 = solve(g)
    u2, r2 = solve(np.roll(g, p, axis=2))
    assert r1["cycles"] == r2["cycles"]
    a = np.roll(u1, p, axis=2)
    assert np.abs(a - u2).max() <= 1e-10 * np.abs(a).max()
    s.close()


def test_periodic_warp_star_kernel_forced(monkeypatch):
    import paper_1808_03595_b200 as pmg
    monkeypatch.setenv("PMG_STAR_W_MIN", "0")
    P = ppair("k423_p4_per_x")
    case = P.case
    s = pmg.Solver(case.k, case.widths, case.p, case.lam, periodic=0b001)
    for l in range(s.nlevels):
        r = P.rand_skel(l)
        rs = s.new_skel(l)
        s.skel_from_grid(l, torch.from_numpy(r).cuda(), rs)
        du = s.new_skel(l)
        s.smooth(l, rs, du)
        g = s.new_grid(l)
        s.skel_to_grid(l, du, g)
        torch.cuda.synchronize()
        assert close(g.cpu().numpy(), P.orc.levels[l].mesh.fill_periodic(P.orc.levels[l].smoother.apply(r)), OP_TOL), l
    s.close()


def test_periodic_invalid_options():
    import paper_1808_03595_b200 as pmg
    case = pi.small_case((3, 2, 2), 4, 0.5)
    with pytest.raises(pmg.PmgError):
        pmg.Solver(case.k, case.widths, 4, 0.5, periodic=0b001)             # odd k_1
    case = pi.small_case((2, 2, 2), 4, 0.0)
    with pytest.raises(pmg.PmgError):
        pmg.Solver(case.k, case.widths, 4, 0.0, periodic=0b111)             # singular fully periodic Poisson
    with pytest.raises(pmg.PmgError):
        pmg.Solver(case.k, case.widths, 4, 1.0, periodic=0b001, neumann=0b000001)
    with pytest.raises(pmg.PmgError):
        pmg.Solver(case.k, case.widths, 4, 1.0, periodic=0b001, smoother=1)
