"""p-multigrid V-cycle and solver for the condensed system (oracle).

P:426-434: p_l = p0 2^l for 0 <= l < L, p_L = p; p0 = 2.  Reading c-10: for a p that
  is not p0 times a power of two, L = ceil(log2(p / p0)).
P:440: the coarse grid solver is "a conjugate gradient solver working in the condensed system at
  p0 = 2".  Reading c-11: Jacobi (exact diag of H_hat_0) preconditioned CG, zero initial guess,
  stopped at ||r|| <= rtol_c ||b||.
P:443-480 Alg. 3 (V-cycle) with nu_pre = nu_post = 1 ("MG") or 2^(L-l).
P:483-506 Alg. 4 (solver): condense, cycle while ||r_hat|| > eps, recover.  Reading c-12: eps =
  rtol ||r_hat_0|| with rtol = 1e-10 (the "reduction by 1e-10" of P:636), zero initial guess.
P:636-641: n_10 and rho = (||r_n|| / ||r_0||)^(1/n).
Reading c-9: the restriction in Alg. 3 (printed J_hat_{l-1}^T) is J_hat_l^T.
"""
import math

import numpy as np

from .mesh import Mesh
from .condensed import CondensedOperator
from .smoother import StarSmoother
from .ecsmoother import ECSmoother
from .transfer import Transfer


def level_degrees(p, p0=2):
    if p < p0:
        raise ValueError("p >= p0 required for a multigrid hierarchy")
    L = 0 if p == p0 else int(math.ceil(math.log2(p / p0) - 1e-12))
    return [p0 * 2 ** l for l in range(L)] + [p]


class Level:
    def __init__(self, k, widths, p, lam, pw, neumann=0, smoother="star", periodic=0):
        """smoother: "star" (vertex stars, Alg. 2) or "element" (element-centred blocks, NEXT-4).
        periodic: bitmask of periodic directions (Mesh; NEXT-3)."""
        self.mesh = Mesh(k, widths, p, neumann=neumann, periodic=periodic)
        if periodic and smoother != "star":
            raise ValueError("periodic directions: vertex-star smoother only")
        self.op = CondensedOperator(self.mesh, lam)
        if smoother not in ("star", "element"):
            raise ValueError("smoother must be 'star' or 'element'")
        self.smoother = StarSmoother(self.op, pw) if smoother == "star" else ECSmoother(self.op, pw)
        d = self.op.diag()
        self.dinv = np.where(self.mesh.free_skel, 1.0 / np.where(d != 0, d, 1.0), 0.0)


def pcg(level, b, rtol, maxit):
    """Jacobi-preconditioned CG on H_hat_0 x = b from x = 0 (reading c-11).  Returns (x, its)."""
    op = level.op
    x = np.zeros_like(b)
    r = b.copy()
    bnorm = math.sqrt(float(r @ r))
    if bnorm == 0.0:
        return x, 0
    z = level.dinv * r
    pv = z.copy()
    rz = float(r @ z)
    for it in range(1, maxit + 1):
        q = op.apply(pv)
        pq = float(pv @ q)
        if not pq > 0.0:
            raise FloatingPointError("CG breakdown: p^T H p <= 0")
        alpha = rz / pq
        x += alpha * pv
        r -= alpha * q
        if math.sqrt(float(r @ r)) <= rtol * bnorm:
            return x, it
        z = level.dinv * r
        rz_new = float(r @ z)
        beta = rz_new / rz
        rz = rz_new
        pv = z + beta * pv
    return x, maxit


class Hierarchy:
    def __init__(self, k, widths, p, lam, p0=2, pw=7, schedule=0, coarse_rtol=1e-4,
                 coarse_maxit=10000, neumann=0, coarse_solver="auto", smoother="star", periodic=0):
        """neumann: face bitmask of homogeneous Neumann faces (Mesh; NEXT-3).
        coarse_solver: "jacobi" (Jacobi-PCG, reading R11), "hmg" (CG preconditioned by the
        h-multigrid V-cycle of oracle/hmg.py, reading R16) or "auto" (hmg iff more than 12288
        elements, some k_d halvable and lambda L_min^2 < 100 -- the rule the GPU library uses)."""
        self.degrees = level_degrees(p, p0)
        self.L = len(self.degrees) - 1
        self.levels = [Level(k, widths, q, lam, pw, neumann, smoother if l > 0 else "star", periodic)
                       for l, q in enumerate(self.degrees)]
        self.transfers = [None] + [Transfer(self.levels[l - 1].mesh, self.levels[l].mesh)
                                   for l in range(1, self.L + 1)]
        self.schedule = schedule
        from . import hmg as _hmg
        if coarse_solver == "auto":
            ne = int(np.prod(k))
            lmin = min(float(np.sum(w)) for w in widths)
            coarse_solver = ("hmg" if (p0 == 2 and ne > 12288 and _hmg.coarsenable(k) and lam * lmin * lmin < 100.0
                                       and not periodic) else "jacobi")
        if coarse_solver == "hmg" and periodic:
            raise ValueError("the h-multigrid coarse solver does not support periodic directions")
        self.coarse_solver = coarse_solver
        self.hmg = _hmg.HMultigrid(k, widths, lam, neumann) if coarse_solver == "hmg" else None
        self.coarse_rtol = coarse_rtol
        self.coarse_maxit = coarse_maxit
        self.coarse_its = []

    def nu(self, l):
        return 1 if self.schedule == 0 else 2 ** (self.L - l)

    def smooth_step(self, l, u, f):
        """u <- u + Smoother(f - H_l u) (Alg. 3 pre/post-smoothing line)."""
        lv = self.levels[l]
        return u + lv.smoother.apply(lv.op.residual(u, f))

    def coarse_solve(self, f0):
        if self.hmg is not None:
            from .hmg import pcg_hmg
            x, its = pcg_hmg(self.levels[0], self.hmg, f0, self.coarse_rtol, self.coarse_maxit)
            self.coarse_its.append(its)
            return x
        x, its = pcg(self.levels[0], f0, self.coarse_rtol, self.coarse_maxit)
        self.coarse_its.append(its)
        return x

    def vcycle(self, u, f):
        """Alg. 3."""
        L = self.L
        if L == 0:
            # reading c-10b: with a single level the "coarse solve" of Alg. 3 acts on the
            # residual equation, u <- u + CG(f - H_0 u), so that Alg. 4 remains a fixpoint
            # iteration (CG restarted from zero every cycle, like the multilevel coarse solve).
            lv = self.levels[0]
            return np.asarray(u) + self.coarse_solve(lv.op.residual(u, f))
        us = [None] * (L + 1)
        fs = [None] * (L + 1)
        us[L] = np.asarray(u, dtype=np.float64).copy()
        fs[L] = np.asarray(f, dtype=np.float64)
        for l in range(L, 0, -1):
            if l != L:
                us[l] = np.zeros(self.levels[l].mesh.ntot)
            for _ in range(self.nu(l)):
                us[l] = self.smooth_step(l, us[l], fs[l])
            r = self.levels[l].op.residual(us[l], fs[l])
            fs[l - 1] = self.transfers[l].restrict(r)
        us[0] = self.coarse_solve(fs[0])
        for l in range(1, L + 1):
            us[l] = us[l] + self.transfers[l].prolong(us[l - 1])
            for _ in range(self.nu(l)):
                us[l] = self.smooth_step(l, us[l], fs[l])
        return us[L]

    def solve(self, F, rtol=1e-10, max_cycles=50):
        """Alg. 4.  Returns (u_full, report dict)."""
        top = self.levels[-1]
        op = top.op
        fhat = op.condense(F)
        u = np.zeros(top.mesh.ntot)
        r = op.residual(u, fhat)
        r0 = math.sqrt(float(r @ r))
        hist = [r0]
        cycles = 0
        rn = r0
        while rn > rtol * r0 and cycles < max_cycles:
            u = self.vcycle(u, fhat)
            r = op.residual(u, fhat)
            rn = math.sqrt(float(r @ r))
            hist.append(rn)
            cycles += 1
        rho = (rn / r0) ** (1.0 / cycles) if cycles and r0 > 0 else 0.0
        u_full = top.mesh.fill_periodic(op.recover(u, F))
        rep = dict(cycles=cycles, r0=r0, r_final=rn, rho=rho, history=hist,
                   converged=bool(rn <= rtol * r0), u_hat=u, f_hat=fhat)
        return u_full, rep

    def solve_ipcg(self, F, rtol=1e-10, max_iters=50):
        """Alg. 5, Krylov-accelerated multigrid, verbatim: inexact preconditioned CG
        (Golub & Ye) with one V-cycle from zero as the preconditioner.  kMG with schedule 0, kvMG
        with schedule 1.  Stopping test as Alg. 4 (reading R12): ||r|| <= rtol ||r_0||.
        Returns (u_full, report dict) like solve()."""
        top = self.levels[-1]
        op = top.op
        fhat = op.condense(F)
        u = np.zeros(top.mesh.ntot)
        r = op.residual(u, fhat)                       # initial residual
        s = r.copy()                                   # ensures beta = 0 on the first iteration
        p = np.zeros_like(r)
        delta = 1.0
        r0 = math.sqrt(float(r @ r))
        hist = [r0]
        its = 0
        rn = r0
        while rn > rtol * r0 and its < max_iters:
            z = self.vcycle(np.zeros_like(r), r)        # preconditioner
            gamma = float(z @ r)
            gamma0 = float(z @ s)
            beta = (gamma - gamma0) / delta
            delta = gamma
            p = beta * p + z                            # update search vector
            q = op.apply(p)                             # effect of p
            alpha = gamma / float(q @ p)                # step width
            s = r.copy()                                # save old residual
            u = u + alpha * p
            r = r - alpha * q
            rn = math.sqrt(float(r @ r))
            hist.append(rn)
            its += 1
        rho = (rn / r0) ** (1.0 / its) if its and r0 > 0 else 0.0
        u_full = top.mesh.fill_periodic(op.recover(u, F))
        rep = dict(cycles=its, r0=r0, r_final=rn, rho=rho, history=hist,
                   converged=bool(rn <= rtol * r0), u_hat=u, f_hat=fhat)
        return u_full, rep
