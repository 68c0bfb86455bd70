"""CPU-side checks of the C ABI: the in-tree library builds/loads and exports every symbol that
include/pmg.h declares; host-only entry points behave; no GPU is touched."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "pmg.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pmg_[a-z_]+)\s*\(", src)))


def _lib():
    import importlib
    path = os.path.join(ROOT, "paper_1808_03595_b200", "libpmg.so")
    if not os.path.exists(path):
        importlib.import_module("paper_1808_03595_b200.build").build()
    return ctypes.CDLL(path)


def test_header_declares_the_north_star_calls():
    names = _declared()
    for want in ("pmg_setup", "pmg_residual", "pmg_smooth", "pmg_restrict", "pmg_prolong",
                 "pmg_vcycle", "pmg_solve", "pmg_condense", "pmg_recover", "pmg_destroy"):
        assert want in names


def test_library_exports_every_declared_symbol():
    lib = _lib()
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_default_options_and_error_string():
    import paper_1808_03595_b200 as pmg
    o = pmg.default_options()
    assert (o.p0, o.weight_degree, o.schedule, o.coarse_maxit, o.nranks) == (2, 7, 0, 10000, 1)
    assert o.coarse_rtol == 1e-4
    lib = _lib()
    lib.pmg_last_error.restype = ctypes.c_char_p
    lib.pmg_destroy.argtypes = [ctypes.c_void_p]
    assert lib.pmg_destroy(None) == -1                      # PMG_EINVAL, message set
    assert b"NULL" in lib.pmg_last_error()


def test_setup_rejects_bad_arguments_before_touching_the_gpu():
    import numpy as np
    import paper_1808_03595_b200 as pmg
    lib = pmg._lib
    for k, w, p, lam in [((2, 2, 2), [np.ones(2)] * 3, 1, 0.0), ((2, 2, 2), [np.ones(2)] * 3, 33, 0.0),
                         ((2, 2, 2), [np.array([1.0, 0.0])] * 3, 4, 0.0), ((2, 2, 2), [np.ones(2)] * 3, 4, -2.0),
                         ((0, 2, 2), [np.ones(1), np.ones(2), np.ones(2)], 4, 0.0),
                         ((2, 2, 2), [np.array([1.0, np.inf])] * 3, 4, 0.0)]:
        ws = [np.ascontiguousarray(x, dtype=np.float64) for x in w]
        ne = (ctypes.c_int * 3)(*k)
        wp = (ctypes.POINTER(ctypes.c_double) * 3)(*[x.ctypes.data_as(ctypes.POINTER(ctypes.c_double)) for x in ws])
        h = ctypes.c_void_p()
        st = lib.pmg_setup(ctypes.byref(h), ne, wp, p, lam, None)
        assert st == pmg.PMG_EINVAL and not h.value, (k, p, lam, st)
        assert lib.pmg_last_error()


def test_smoother_option_validated_before_touching_the_gpu():
    """smoother: 0 vertex stars (default), 1 element-centred blocks (NEXT-4): p <= 16, one rank."""
    import numpy as np
    import paper_1808_03595_b200 as pmg
    lib = pmg._lib
    assert pmg.default_options().smoother == 0
    ws = [np.ones(2)] * 3
    ne = (ctypes.c_int * 3)(2, 2, 2)
    wp = (ctypes.POINTER(ctypes.c_double) * 3)(*[x.ctypes.data_as(ctypes.POINTER(ctypes.c_double)) for x in ws])
    for p, sm, nranks in [(4, 2, 1), (4, -1, 1), (20, 1, 1), (4, 1, 2)]:
        o = pmg.default_options()
        o.smoother, o.nranks = sm, nranks
        h = ctypes.c_void_p()
        assert lib.pmg_setup(ctypes.byref(h), ne, wp, p, 0.0, ctypes.byref(o)) == pmg.PMG_EINVAL
        assert not h.value and b"smoother" in lib.pmg_last_error()
