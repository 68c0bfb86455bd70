"""Thin Python binding of the B200 p-multigrid C ABI (include/pmg.h).

Argument marshalling only: every step of the method runs in the CUDA kernels of libpmg.so.
Vectors are torch CUDA float64 tensors (device memory, caller-owned); torch is used for memory,
streams and process groups only.  There is no CPU fallback: importing this package without the
built library raises ImportError.
"""
import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PMG_LIB") or os.path.join(HERE, "libpmg.so")   # PMG_LIB: experiment builds only

if not os.path.exists(LIB_PATH):
    raise ImportError("libpmg.so not built: run `python paper_1808_03595_b200/build.py` "
                      "(or __graft_entry__.build()); there is no fallback implementation")

import torch  # noqa: E402,F401  (load torch's NCCL before libpmg.so resolves libnccl.so.2)

_lib = ctypes.CDLL(LIB_PATH)

PMG_OK, PMG_EINVAL, PMG_ECUDA, PMG_ENCCL, PMG_ENOCONV, PMG_EBREAKDOWN, PMG_ENOMEM = 0, -1, -2, -3, -4, -5, -6
_STATUS = {0: "PMG_OK", -1: "PMG_EINVAL", -2: "PMG_ECUDA", -3: "PMG_ENCCL", -4: "PMG_ENOCONV",
           -5: "PMG_EBREAKDOWN", -6: "PMG_ENOMEM"}


class PmgError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__("%s: %s" % (_STATUS.get(status, status), msg))
        self.status = status


class Options(ctypes.Structure):
    _fields_ = [("p0", ctypes.c_int), ("weight_degree", ctypes.c_int), ("schedule", ctypes.c_int),
                ("neumann", ctypes.c_int), ("periodic", ctypes.c_int), ("solver", ctypes.c_int),
                ("smoother", ctypes.c_int),
                ("coarse_rtol", ctypes.c_double), ("coarse_maxit", ctypes.c_int),
                ("coarse_check", ctypes.c_int), ("coarse_solver", ctypes.c_int),
                ("rank", ctypes.c_int), ("nranks", ctypes.c_int),
                ("nccl_id", ctypes.c_void_p), ("loopback", ctypes.c_void_p), ("stream", ctypes.c_void_p)]


class Slab(ctypes.Structure):
    """pmg_slab: z-slab plan of one rank (include/pmg.h)."""
    _fields_ = [("z0", ctypes.c_int), ("z1", ctypes.c_int), ("zb", ctypes.c_int), ("nplanes", ctypes.c_int),
                ("own_lo", ctypes.c_int), ("own_hi", ctypes.c_int), ("lower", ctypes.c_int), ("upper", ctypes.c_int)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class Report(ctypes.Structure):
    _fields_ = [("cycles", ctypes.c_int), ("converged", ctypes.c_int), ("r0", ctypes.c_double),
                ("r_final", ctypes.c_double), ("rho", ctypes.c_double), ("coarse_iters", ctypes.c_int),
                ("history", ctypes.POINTER(ctypes.c_double)), ("history_cap", ctypes.c_int),
                ("t_condense", ctypes.c_double), ("t_cycles", ctypes.c_double), ("t_coarse", ctypes.c_double),
                ("t_recover", ctypes.c_double)]


_P = ctypes.c_void_p
_lib.pmg_default_options.argtypes = [ctypes.POINTER(Options)]
_lib.pmg_default_options.restype = None
_lib.pmg_last_error.restype = ctypes.c_char_p
_lib.pmg_setup.argtypes = [ctypes.POINTER(_P), ctypes.POINTER(ctypes.c_int),
                           ctypes.POINTER(ctypes.POINTER(ctypes.c_double)), ctypes.c_int, ctypes.c_double,
                           ctypes.POINTER(Options)]
_lib.pmg_destroy.argtypes = [_P]
_lib.pmg_num_levels.argtypes = [_P]
_lib.pmg_level_info.argtypes = [_P, ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_longlong),
                                ctypes.POINTER(ctypes.c_longlong)]
_lib.pmg_grid_coords.argtypes = [_P, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_double)]
_lib.pmg_residual.argtypes = [_P, ctypes.c_int, _P, _P, _P]
_lib.pmg_smooth.argtypes = [_P, ctypes.c_int, _P, _P]
_lib.pmg_restrict.argtypes = [_P, ctypes.c_int, _P, _P]
_lib.pmg_prolong.argtypes = [_P, ctypes.c_int, _P, _P]
_lib.pmg_vcycle.argtypes = [_P, _P, _P]
_lib.pmg_condense.argtypes = [_P, _P, _P]
_lib.pmg_recover.argtypes = [_P, _P, _P, _P]
_lib.pmg_solve.argtypes = [_P, _P, _P, ctypes.c_double, ctypes.c_int, ctypes.POINTER(Report)]
_lib.pmg_solve_host.argtypes = [_P, _P, _P, ctypes.c_double, ctypes.c_int, ctypes.POINTER(Report)]
_lib.pmg_weak_rhs.argtypes = [_P, _P, _P]
_lib.pmg_skel_from_grid.argtypes = [_P, ctypes.c_int, _P, _P]
_lib.pmg_skel_to_grid.argtypes = [_P, ctypes.c_int, _P, _P]
_lib.pmg_norm.argtypes = [_P, ctypes.c_int, _P, ctypes.POINTER(ctypes.c_double)]
_lib.pmg_launch_count.argtypes = [_P]
_lib.pmg_launch_count.restype = ctypes.c_longlong
_lib.pmg_timing_enable.argtypes = [_P, ctypes.c_int]
_lib.pmg_timing_read.argtypes = [_P, ctypes.c_int, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_longlong)]
_lib.pmg_timing_enable.restype = ctypes.c_int
_lib.pmg_slab_plan.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(Slab)]
_lib.pmg_slab_plan.restype = ctypes.c_int
_lib.pmg_slab_info.argtypes = [_P, ctypes.POINTER(Slab)]
_lib.pmg_nccl_unique_id.argtypes = [_P]
_lib.pmg_loopback_create.argtypes = [ctypes.c_int]
_lib.pmg_loopback_create.restype = _P
_lib.pmg_loopback_destroy.argtypes = [_P]
_lib.pmg_loopback_destroy.restype = None
_lib.pmg_timing_read.restype = ctypes.c_int
for _name in ("pmg_setup", "pmg_destroy", "pmg_level_info", "pmg_grid_coords", "pmg_residual", "pmg_smooth",
              "pmg_restrict", "pmg_prolong", "pmg_vcycle", "pmg_condense", "pmg_recover", "pmg_solve",
              "pmg_solve_host", "pmg_weak_rhs", "pmg_skel_from_grid", "pmg_skel_to_grid", "pmg_norm",
              "pmg_num_levels", "pmg_slab_info", "pmg_nccl_unique_id"):
    getattr(_lib, _name).restype = ctypes.c_int


def _check(status, allow=()):
    if status != PMG_OK and status not in allow:
        raise PmgError(status, _lib.pmg_last_error().decode())
    return status


def _ptr(t):
    """Device pointer of a CUDA float64 contiguous tensor (or None)."""
    if t is None:
        return None
    if not t.is_cuda or t.dtype.itemsize != 8 or not t.is_contiguous():
        raise TypeError("expected a contiguous CUDA float64 tensor")
    return ctypes.c_void_p(t.data_ptr())


def slab_plan(k3, nranks, rank):
    """z-slab plan of `rank` (pure host arithmetic of the library; no GPU needed)."""
    sl = Slab()
    if _lib.pmg_slab_plan(int(k3), int(nranks), int(rank), ctypes.byref(sl)) != 0:
        raise PmgError(PMG_EINVAL, "invalid slab plan arguments")
    return sl.as_dict()


def nccl_unique_id():
    """128-byte ncclUniqueId (bytes) for pmg_options.nccl_id; create on rank 0 and broadcast."""
    buf = ctypes.create_string_buffer(128)
    _check(_lib.pmg_nccl_unique_id(ctypes.cast(buf, _P)))
    return buf.raw


class Loopback:
    """Hub shared by the contexts of one process that emulate nranks ranks (correctness tests)."""

    def __init__(self, nranks):
        self.h = _lib.pmg_loopback_create(int(nranks))
        if not self.h:
            raise PmgError(PMG_EINVAL, "pmg_loopback_create failed")

    def close(self):
        if self.h:
            _lib.pmg_loopback_destroy(self.h)
            self.h = None


def default_options():
    o = Options()
    _lib.pmg_default_options(ctypes.byref(o))
    return o


class Solver:
    """One pmg context: the level hierarchy for (k, widths, p, lambda) on the current device."""

    def __init__(self, k, widths, p, lam, p0=2, schedule=0, coarse_rtol=1e-4, coarse_maxit=10000,
                 coarse_check=8, stream=None, rank=0, nranks=1, nccl_id=None, loopback=None, solver=0,
                 neumann=0, coarse_solver=0, smoother=0, periodic=0):
        """solver 0: MG fixpoint iteration (Alg. 4); 1: Krylov-accelerated MG (ipCG, Alg. 5).
        neumann: face bitmask of homogeneous Neumann faces (bit 2d / 2d+1: low / high face of d).
        periodic: bitmask of periodic directions (bit d), k_d even.
        smoother 0: vertex stars (Alg. 2); 1: element-centred 3x3x3 blocks (NEXT-4)."""
        import numpy as np
        import torch
        o = default_options()
        o.p0, o.schedule, o.coarse_rtol, o.coarse_maxit, o.coarse_check = p0, schedule, coarse_rtol, coarse_maxit, coarse_check
        o.rank, o.nranks = int(rank), int(nranks)
        o.solver = int(solver)
        o.neumann = int(neumann)
        o.periodic = int(periodic)
        o.coarse_solver = int(coarse_solver)
        o.smoother = int(smoother)
        self._nccl_buf = None
        if nccl_id is not None:
            self._nccl_buf = ctypes.create_string_buffer(bytes(nccl_id), 128)
            o.nccl_id = ctypes.cast(self._nccl_buf, _P)
        if loopback is not None:
            o.loopback = loopback.h
        if stream is None:
            stream = torch.cuda.current_stream()
        self.stream = stream
        o.stream = ctypes.c_void_p(stream.cuda_stream)
        self.k = tuple(int(v) for v in k)
        self._w = [np.ascontiguousarray(np.asarray(w, dtype=np.float64)) for w in widths]
        ne = (ctypes.c_int * 3)(*self.k)
        wp = (ctypes.POINTER(ctypes.c_double) * 3)(*[w.ctypes.data_as(ctypes.POINTER(ctypes.c_double)) for w in self._w])
        h = _P()
        _check(_lib.pmg_setup(ctypes.byref(h), ne, wp, int(p), float(lam), ctypes.byref(o)))
        self._h = h
        self.p, self.lam = int(p), float(lam)
        self.nlevels = _lib.pmg_num_levels(h)
        self.rank, self.nranks = int(rank), int(nranks)
        sl = Slab()
        _check(_lib.pmg_slab_info(h, ctypes.byref(sl)))
        self.slab = sl.as_dict()

    def close(self):
        if getattr(self, "_h", None):
            _lib.pmg_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- geometry
    def level_info(self, level):
        d, ns, ng = ctypes.c_int(), ctypes.c_longlong(), ctypes.c_longlong()
        _check(_lib.pmg_level_info(self._h, level, ctypes.byref(d), ctypes.byref(ns), ctypes.byref(ng)))
        return d.value, ns.value, ng.value

    def grid_coords(self, level, d):
        import numpy as np
        deg, _, _ = self.level_info(level)
        nel = self.k[d] if d < 2 else self.slab["z1"] - self.slab["z0"]   # z: this rank's slab
        x = np.zeros(nel * deg + 1)
        _check(_lib.pmg_grid_coords(self._h, level, d, x.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
        return x

    def new_skel(self, level):
        import torch
        return torch.zeros(self.level_info(level)[1], dtype=torch.float64, device="cuda")

    def new_grid(self, level=None):
        import torch
        level = self.nlevels - 1 if level is None else level
        return torch.zeros(self.level_info(level)[2], dtype=torch.float64, device="cuda")

    # ---- operators (stream-ordered, asynchronous)
    def residual(self, level, u, f, r):
        _check(_lib.pmg_residual(self._h, level, _ptr(u), _ptr(f), _ptr(r)))

    def smooth(self, level, r, u):
        _check(_lib.pmg_smooth(self._h, level, _ptr(r), _ptr(u)))

    def restrict(self, level, r_fine, f_coarse):
        _check(_lib.pmg_restrict(self._h, level, _ptr(r_fine), _ptr(f_coarse)))

    def prolong(self, level, u_coarse, u_fine):
        _check(_lib.pmg_prolong(self._h, level, _ptr(u_coarse), _ptr(u_fine)))

    def vcycle(self, u, f):
        _check(_lib.pmg_vcycle(self._h, _ptr(u), _ptr(f)))

    def condense(self, F, fhat):
        _check(_lib.pmg_condense(self._h, _ptr(F), _ptr(fhat)))

    def recover(self, uhat, F, ufull):
        _check(_lib.pmg_recover(self._h, _ptr(uhat), _ptr(F), _ptr(ufull)))

    def weak_rhs(self, f, F):
        _check(_lib.pmg_weak_rhs(self._h, _ptr(f), _ptr(F)))

    def skel_from_grid(self, level, grid, skel):
        _check(_lib.pmg_skel_from_grid(self._h, level, _ptr(grid), _ptr(skel)))

    def skel_to_grid(self, level, skel, grid):
        _check(_lib.pmg_skel_to_grid(self._h, level, _ptr(skel), _ptr(grid)))

    def norm(self, level, x):
        out = ctypes.c_double()
        _check(_lib.pmg_norm(self._h, level, _ptr(x), ctypes.byref(out)))
        return out.value

    def _report(self, rep, hist, status):
        return dict(cycles=rep.cycles, converged=bool(rep.converged), r0=rep.r0, r_final=rep.r_final,
                    rho=rep.rho, coarse_iters=rep.coarse_iters,
                    history=list(hist[:rep.cycles + 1]), status=status,
                    t_condense=rep.t_condense, t_cycles=rep.t_cycles, t_coarse=rep.t_coarse, t_recover=rep.t_recover)

    def solve(self, F, u, rtol=1e-10, max_cycles=50):
        hist = (ctypes.c_double * (max_cycles + 1))()
        rep = Report(history=hist, history_cap=max_cycles + 1)
        st = _check(_lib.pmg_solve(self._h, _ptr(F), _ptr(u), rtol, max_cycles, ctypes.byref(rep)),
                    allow=(PMG_ENOCONV,))
        return self._report(rep, hist, st)

    def solve_host(self, F_host, u_host, rtol=1e-10, max_cycles=50):
        """F_host, u_host: host float64 buffers (numpy arrays or pinned CPU tensors)."""
        hist = (ctypes.c_double * (max_cycles + 1))()
        rep = Report(history=hist, history_cap=max_cycles + 1)

        def hp(a):
            if hasattr(a, "data_ptr"):
                return ctypes.c_void_p(a.data_ptr())
            return ctypes.c_void_p(a.ctypes.data)
        st = _check(_lib.pmg_solve_host(self._h, hp(F_host), hp(u_host), rtol, max_cycles, ctypes.byref(rep)),
                    allow=(PMG_ENOCONV,))
        return self._report(rep, hist, st)

    def launch_count(self):
        return _lib.pmg_launch_count(self._h)

    def timing_enable(self, on=True):
        _check(_lib.pmg_timing_enable(self._h, 1 if on else 0))

    def timing_read(self, kind):
        """(total_ms, count); kind 0/1: smoother sweep / residual on the finest level,
        2/3: on all levels."""
        ms, n = ctypes.c_double(), ctypes.c_longlong()
        _check(_lib.pmg_timing_read(self._h, kind, ctypes.byref(ms), ctypes.byref(n)))
        return ms.value, n.value


def lib_path():
    return LIB_PATH
