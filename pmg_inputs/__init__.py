"""Seeded synthetic inputs shared by the oracle side and the CUDA side of every test/bench.

This module holds NO arithmetic of the method: it defines the problem (mesh widths, lambda,
degree) of each BASELINE.json config and draws the nodal right-hand side f from a
counter-based generator.  Node coordinates are passed IN by the caller (each side computes its
own GLL grid), so nothing here depends on either implementation.

Generator:  global node id g = i1 + N1 (i2 + N2 i3), N_d = k_d p + 1;
  x = SplitMix64(seed * 2^40 + g);  U = ((x >> 11) * 2^-53) * 2 - 1  in [-1, 1);
  N(0,1) by Box-Muller from the uniforms of ids 2g and 2g+1.
"""
import math
from dataclasses import dataclass, field

import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x):
    """SplitMix64 output function applied to state x + golden gamma (Vigna's reference:
    the first output of a generator seeded with 0 is 0xE220A8397B1DCDAF)."""
    with np.errstate(over="ignore"):
        z = np.asarray(x, dtype=np.uint64) + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def uniform_pm1(seed, ids):
    x = splitmix64(np.uint64(seed) * np.uint64(1 << 40) + np.asarray(ids, dtype=np.uint64))
    return (x >> np.uint64(11)).astype(np.float64) * (2.0 ** -53) * 2.0 - 1.0


def normal(seed, ids):
    ids = np.asarray(ids, dtype=np.uint64)
    u1 = 0.5 * (uniform_pm1(seed, 2 * ids) + 1.0)          # [0, 1)
    u2 = 0.5 * (uniform_pm1(seed, 2 * ids + 1) + 1.0)
    u1 = np.where(u1 <= 0.0, 2.0 ** -53, u1)
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)


@dataclass
class Case:
    """One problem: k elements per direction, widths per direction, degree p, lambda and the
    nodal right-hand side recipe."""
    name: str
    k: tuple
    widths: list
    p: int
    lam: float
    f_kind: str            # "uniform" | "normal" | "sin3" | "sin3_noise" | "sin3_lambda"
    seed: int = 0
    amp: float = 1.0
    noise: float = 0.0
    origin: tuple = (0.0, 0.0, 0.0)
    meta: dict = field(default_factory=dict)

    @property
    def N(self):
        return tuple(kd * self.p + 1 for kd in self.k)

    @property
    def n_dof(self):
        """Unknowns n_e p^3 (the paper's convention)."""
        return self.k[0] * self.k[1] * self.k[2] * self.p ** 3

    def f_nodal(self, coords, i3_offset=0):
        """Nodal f on the global grid (flat, x1 fastest) given the three 1-D coordinate arrays.
        A z-slab passes its own x3 nodes and the global index of its first plane (i3_offset):
        the values are those of the undivided grid on those planes."""
        N1, N2, N3 = self.N
        n3 = len(coords[2])
        g = np.arange(N1 * N2 * n3, dtype=np.uint64) + np.uint64(N1 * N2 * int(i3_offset))
        if self.f_kind == "uniform":
            return uniform_pm1(self.seed, g)
        if self.f_kind == "normal":
            return normal(self.seed, g)
        x1, x2, x3 = [np.asarray(c, dtype=np.float64) for c in coords]
        s = (np.sin(x3)[:, None, None] * np.sin(x2)[None, :, None] * np.sin(x1)[None, None, :]).ravel()
        f = self.amp * s
        if self.noise:
            f = f + self.noise * uniform_pm1(self.seed, g)
        return f


def uniform_widths(k, length):
    return [np.full(kd, L / kd) for kd, L in zip(k, length)]


def geometric_widths(k, length, ratio):
    """One-sided geometric widths h_i = h_0 ratio^i, i = 0..k-1, summing to ``length``
    (reading c-13 for the paper's 'constant expansion factor')."""
    r = ratio ** np.arange(k)
    return length * r / r.sum()


TWO_PI = 2.0 * math.pi


def config(i, p=None, n_gpu=1):
    """BASELINE.json configs[i-1] (1-based)."""
    if i == 1:
        k = (4, 4, 4)
        return Case("cfg1_helmholtz_4x4x4_p4", k, uniform_widths(k, (TWO_PI,) * 3), 4, 1.0,
                    "sin3", seed=0, amp=3.0, noise=1e-3)
    if i == 2:
        k = (16, 16, 16)
        return Case("cfg2_poisson_16x16x16_p8", k, uniform_widths(k, (1.0,) * 3), 8, 0.0,
                    "uniform", seed=1)
    if i == 3:
        p = 8 if p is None else p
        kk = int(round(256 / p))
        k = (kk, kk, kk)
        return Case("cfg3_sweep_%dx%dx%d_p%d" % (kk, kk, kk, p), k, uniform_widths(k, (TWO_PI,) * 3),
                    p, 0.0, "normal", seed=2)
    if i == 4:
        k = (32, 32, 32)
        w = [geometric_widths(32, TWO_PI, 1.1), np.full(32, TWO_PI / 32), np.full(32, TWO_PI / 32)]
        return Case("cfg4_helmholtz_stretched_32x32x32_p16", k, w, 16, 100.0, "sin3", seed=3,
                    amp=1.0)
    if i == 5:
        k = (64, 64, 8 * n_gpu)
        return Case("cfg5_poisson_64x64x%d_p16" % (8 * n_gpu), k,
                    uniform_widths(k, (1.0, 1.0, n_gpu / 8.0)), 16, 0.0, "uniform", seed=4)
    raise ValueError("configs are 1..5")


def small_case(k=(3, 3, 3), p=4, lam=0.0, seed=7, stretch=None, kind="uniform"):
    """Small seeded cases for parity tests (oracle finishes in seconds)."""
    if stretch is None:
        w = uniform_widths(k, (1.0,) * 3)
    else:
        w = [geometric_widths(k[0], 1.0, stretch), np.full(k[1], 1.3 / k[1]),
             geometric_widths(k[2], 0.8, 1.0 / stretch)]
    return Case("small_%dx%dx%d_p%d" % (k + (p,)), tuple(k), w, p, lam, kind, seed=seed)
