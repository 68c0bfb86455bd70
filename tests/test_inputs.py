"""The seeded input generator (shared by both sides; holds no method arithmetic)."""
import numpy as np

import pmg_inputs as pi


def test_splitmix64_reference_value():
    # Vigna's splitmix64.c: the first output of a generator with state 0 is 0xE220A8397B1DCDAF
    assert int(pi.splitmix64(np.uint64(0))) == 0xE220A8397B1DCDAF


def test_uniform_range_and_determinism():
    u = pi.uniform_pm1(1, np.arange(100000))
    assert u.min() >= -1 and u.max() < 1 and abs(u.mean()) < 0.01
    assert np.array_equal(u, pi.uniform_pm1(1, np.arange(100000)))
    assert not np.array_equal(u, pi.uniform_pm1(2, np.arange(100000)))
    z = pi.normal(2, np.arange(200000))
    assert abs(z.mean()) < 0.01 and abs(z.std() - 1) < 0.01


def test_configs():
    c = pi.config(2)
    assert c.n_dof == 16 ** 3 * 8 ** 3 and c.p == 8 and c.lam == 0.0
    c4 = pi.config(4)
    assert abs(c4.widths[0].sum() - 2 * np.pi) < 1e-12
    assert abs(c4.widths[0][-1] / c4.widths[0][0] - 1.1 ** 31) < 1e-9
    for p in (2, 4, 8, 12, 16, 24, 32):
        c3 = pi.config(3, p)
        assert c3.k[0] == round(256 / p)
