"""Thin ctypes binding of ``include/sip.h`` (argument marshalling only).

Every step of the PARSDMM path runs in the CUDA kernels of ``libsip.so``;
this module only converts Python objects to pointers and sizes.  There is no
CPU fallback: importing it without the built library raises.

Arrays: torch tensors (CUDA or CPU) or numpy arrays (host).  Vectors are
passed as pointers; the library detects host vs device memory.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# SIP_LIBPATH: another in-tree build of the same library (A/B timing tools)
_LIBPATH = os.environ.get("SIP_LIBPATH") or os.path.join(_HERE, "libsip.so")

SIP_OK = 0
SIP_NOT_CONVERGED = 1
SIP_MAX_SETS = 16
OPS = {"I": 0, "IDENTITY": 0, "DZ": 1, "DY": 2, "DX": 3, "TV": 4, "BLUR_MASK": 5}
KINDS = {"bounds": 0, "l1": 1, "l2": 2, "annulus": 3, "card": 4, "rank": 5, "nuclear": 6, "dct_l1": 7, "haar_l1": 8}
DTYPES = {"f32": 0, "f64": 1}


class SipError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"sip status {status}: {msg}")
        self.status = status


class SetParams(C.Structure):
    _fields_ = [
        ("lo", C.c_double), ("hi", C.c_double),
        ("lo_vec", C.c_void_p), ("hi_vec", C.c_void_p),
        ("sigma", C.c_double), ("sigma_lo", C.c_double), ("sigma_hi", C.c_double),
        ("k", C.c_int64), ("k_frac", C.c_double), ("relative", C.c_int),
        ("app_mode", C.c_int),
    ]


class BlurMaskDesc(C.Structure):
    _fields_ = [("kernel", C.c_void_p), ("kh", C.c_int), ("kw", C.c_int), ("mask", C.c_void_p)]


class CommDesc(C.Structure):
    _fields_ = [("nranks", C.c_int), ("rank", C.c_int), ("nccl_unique_id", C.c_void_p)]


class Result(C.Structure):
    _fields_ = [
        ("iterations", C.c_int), ("cg_iterations", C.c_int), ("converged", C.c_int),
        ("breakdown", C.c_int), ("r_evol", C.c_double), ("ms", C.c_double),
        ("r_feas", C.c_double * SIP_MAX_SETS), ("rho", C.c_double * (SIP_MAX_SETS + 1)),
        ("gamma", C.c_double * (SIP_MAX_SETS + 1)),
    ]


EXPORTS = [
    "sip_comm_unique_id", "sip_create_grid", "sip_add_set", "sip_set_option", "sip_project",
    "sip_project_multilevel", "sip_destroy", "sip_status_string", "sip_last_error",
    "sip_apply_op", "sip_apply_system", "sip_cg", "sip_project_set", "sip_get_state",
    "sip_get_log", "sip_get_support_log", "sip_dykstra", "sip_get_sizes", "sip_get_launch_count", "sip_get_profile", "sip_slab",
]
KERNEL_KINDS = ["blur", "rhs", "cg1", "cg2", "pass1", "select", "tiecount", "pass2", "control", "comm", "cgx", "fiber",
                "svd", "dct"]

_lib = None


def lib():
    """Load libsip.so (must be built; no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIBPATH):
            raise ImportError(
                f"{_LIBPATH} is missing: build it with `python -m paper_1902_09699_b200.build` "
                "(there is no CPU fallback)")
        L = C.CDLL(_LIBPATH)
        L.sip_status_string.restype = C.c_char_p
        L.sip_last_error.restype = C.c_char_p
        L.sip_destroy.restype = None
        L.sip_create_grid.argtypes = [C.c_int, C.POINTER(C.c_int64), C.POINTER(C.c_double), C.c_int,
                                      C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p)]
        L.sip_add_set.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.POINTER(SetParams),
                                  C.POINTER(C.c_int)]
        L.sip_set_option.argtypes = [C.c_void_p, C.c_char_p, C.c_double]
        L.sip_project.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_double,
                                  C.POINTER(Result)]
        L.sip_project_multilevel.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int,
                                             C.c_int, C.c_double, C.POINTER(Result)]
        L.sip_destroy.argtypes = [C.c_void_p]
        L.sip_last_error.argtypes = [C.c_void_p]
        L.sip_apply_op.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
        L.sip_apply_system.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.c_void_p, C.c_void_p]
        L.sip_cg.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.c_void_p, C.c_void_p, C.c_int,
                             C.c_int, C.POINTER(C.c_int)]
        L.sip_project_set.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
        L.sip_get_state.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p]
        L.sip_get_log.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                  C.c_void_p, C.c_void_p, C.c_void_p]
        L.sip_get_sizes.argtypes = [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int64), C.c_int,
                                    C.POINTER(C.c_int64)]
        L.sip_get_launch_count.argtypes = [C.c_void_p, C.POINTER(C.c_int64)]
        L.sip_get_profile.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
        L.sip_slab.argtypes = [C.c_int64, C.c_int, C.c_int, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.sip_comm_unique_id.argtypes = [C.c_void_p]
        L.sip_dykstra.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_double, C.c_int, C.c_double,
                                  C.c_void_p]
        _lib = L
    return _lib


def _ptr(a):
    """pointer of a torch tensor or numpy array (must be contiguous)"""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        if not a.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return C.c_void_p(a.data_ptr())
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return C.c_void_p(a.ctypes.data)
    raise TypeError(f"unsupported array type {type(a)}")


def _f64_host(a):
    if a is None:
        return None
    if hasattr(a, "detach"):
        a = a.detach().cpu().numpy()
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64).ravel())


def _current_stream():
    try:
        import torch
        if torch.cuda.is_available():
            return C.c_void_p(torch.cuda.current_stream().cuda_stream)
    except Exception:  # pragma: no cover
        pass
    return C.c_void_p(0)


_NP_DT = {"f32": "float32", "f64": "float64"}


class DykstraLog(C.Structure):
    _fields_ = [("iterations", C.c_int), ("cg_max", C.POINTER(C.c_int)), ("l1_proj", C.POINTER(C.c_int)),
                ("inner_iters", C.POINTER(C.c_int)), ("r_feas", C.POINTER(C.c_double)),
                ("r_evol", C.POINTER(C.c_double))]


class Grid:
    """A PARSDMM problem on a 2D/3D grid (compgrid + set definitions)."""

    def __init__(self, shape, h=None, dtype="f32", stream=None, comm=None):
        self.shape = tuple(int(s) for s in shape)
        self.ndim = len(self.shape)
        self.dtype = dtype
        n = (C.c_int64 * self.ndim)(*self.shape)
        hh = (C.c_double * self.ndim)(*(h or [1.0] * self.ndim))
        handle = C.c_void_p()
        st = stream if stream is not None else _current_stream()
        cd = None
        if comm is not None:
            self._uid = comm["uid"]
            cd = C.byref(CommDesc(comm["nranks"], comm["rank"], _ptr(comm["uid"])))
        s = lib().sip_create_grid(self.ndim, n, hh, DTYPES[dtype], cd, st, C.byref(handle))
        if s != SIP_OK:
            raise SipError(s, lib().sip_status_string(s).decode())
        self.h = handle
        self.sets = []
        self._keep = []

    # -- helpers
    def _check(self, s, allow=(SIP_OK,)):
        if s not in allow:
            raise SipError(s, (lib().sip_last_error(self.h) or b"").decode() or
                           lib().sip_status_string(s).decode())
        return s

    def close(self):
        if getattr(self, "h", None):
            lib().sip_destroy(self.h)
            self.h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    @property
    def N(self):
        return int(np.prod(self.shape))

    def n_local(self):
        """grid points of this rank's slab (the whole grid on one rank)"""
        n = C.c_int64(0)
        self._check(lib().sip_get_sizes(self.h, None, C.byref(n), -1, None))
        return n.value

    def _buf(self, a, n, what):
        """validate a buffer handed to the C ABI: element count, dtype, layout
        (the library copies n * sizeof(dtype) bytes through the pointer)"""
        if a is None:
            raise ValueError(f"{what}: buffer is None")
        want = _NP_DT[self.dtype]
        if hasattr(a, "data_ptr"):
            dt = str(a.dtype).replace("torch.", "")
            numel = a.numel()
            if a.is_cuda:
                import torch
                if a.device.index != torch.cuda.current_device():
                    raise ValueError(f"{what}: tensor on {a.device}, grid on cuda:{torch.cuda.current_device()}")
        elif isinstance(a, np.ndarray):
            dt, numel = a.dtype.name, a.size
        else:
            raise TypeError(f"{what}: unsupported array type {type(a)}")
        if dt != want:
            raise ValueError(f"{what}: dtype {dt}, the grid is {want}")
        if numel != n:
            raise ValueError(f"{what}: {numel} elements, expected {n}")
        return _ptr(a)

    def set_option(self, key, value):
        self._check(lib().sip_set_option(self.h, key.encode(), float(value)))

    def add_set(self, sd):
        """sd: an object with the fields of sip_inputs.SetDef"""
        prm = SetParams()
        prm.lo = float(sd.lo)
        prm.hi = float(sd.hi)
        lo = _f64_host(getattr(sd, "lo_vec", None))
        hi = _f64_host(getattr(sd, "hi_vec", None))
        self._keep += [lo, hi]
        prm.lo_vec = _ptr(lo)
        prm.hi_vec = _ptr(hi)
        prm.sigma = float(sd.sigma)
        prm.sigma_lo = float(sd.sigma_lo)
        prm.sigma_hi = float(sd.sigma_hi)
        prm.k = int(sd.k)
        prm.k_frac = float(sd.k_frac)
        prm.relative = int(bool(sd.relative))
        prm.app_mode = {"": 0, "x": 1, "z": 2}[getattr(sd, "app_mode", "") or ""]
        desc = None
        if sd.op == "BLUR_MASK":
            K = np.ascontiguousarray(sd.kernel, dtype=np.float64)
            mk = np.ascontiguousarray(sd.mask, dtype=np.uint8).ravel()
            self._keep += [K, mk]
            desc = C.byref(BlurMaskDesc(_ptr(K), K.shape[0], K.shape[1], _ptr(mk)))
        sid = C.c_int(-1)
        self._check(lib().sip_add_set(self.h, OPS[sd.op], desc, KINDS[sd.kind], C.byref(prm),
                                      C.byref(sid)))
        self.sets.append(sd)
        return sid.value

    def project(self, m, x, max_iter=200, tol=1e-3):
        r = Result()
        s = self._check(lib().sip_project(self.h, self._buf(m, self.n_local(), "m"), self._buf(x, self.n_local(), "x"), int(max_iter), float(tol),
                                          C.byref(r)), (SIP_OK, SIP_NOT_CONVERGED))
        return _res(r, len(self.sets)), s

    def project_multilevel(self, m, x, n_levels, max_iter=200, tol=1e-3):
        rs = (Result * n_levels)()
        s = self._check(lib().sip_project_multilevel(self.h, self._buf(m, self.n_local(), "m"), self._buf(x, self.n_local(), "x"), int(n_levels), 2,
                                                     int(max_iter), float(tol), rs),
                        (SIP_OK, SIP_NOT_CONVERGED))
        return [_res(rs[l], len(self.sets)) for l in range(n_levels)], s

    def m_len(self, set_id):
        mm = C.c_int64(0)
        self._check(lib().sip_get_sizes(self.h, None, None, int(set_id), C.byref(mm)))
        return mm.value

    def apply_op(self, set_id, x, y):
        self._check(lib().sip_apply_op(self.h, int(set_id), self._buf(x, self.N, "x"),
                                         self._buf(y, self.m_len(set_id), "y")))

    def apply_system(self, rho, p, q):
        r = (C.c_double * len(rho))(*[float(v) for v in rho])
        self._check(lib().sip_apply_system(self.h, r, self._buf(p, self.N, "p"), self._buf(q, self.N, "q")))

    def cg(self, rho, b, x, n_cg, eq25=True):
        r = (C.c_double * len(rho))(*[float(v) for v in rho])
        it = C.c_int(0)
        self._check(lib().sip_cg(self.h, r, self._buf(b, self.N, "b"), self._buf(x, self.N, "x"), int(n_cg), int(bool(eq25)), C.byref(it)))
        return it.value

    def project_set(self, set_id, w, y):
        self._check(lib().sip_project_set(self.h, int(set_id), self._buf(w, self.m_len(set_id), "w"),
                                              self._buf(y, self.m_len(set_id), "y")))

    def get_state(self, set_id, which, out):
        self._check(lib().sip_get_state(self.h, int(set_id), int(which),
                                           self._buf(out, self.m_len(set_id), "out")))

    def get_log(self, max_iter):
        P = len(self.sets) + 1
        p = len(self.sets)
        cg = np.zeros(max_iter, dtype=np.int32)
        br = np.zeros(max_iter * P, dtype=np.int32)
        rt = np.zeros(max_iter * P)
        gt = np.zeros(max_iter * P)
        ft = np.zeros(max(1, max_iter * p))
        et = np.zeros(max_iter)
        self._check(lib().sip_get_log(self.h, int(max_iter), _ptr(cg), _ptr(br), _ptr(rt), _ptr(gt),
                                      _ptr(ft), _ptr(et)))
        return dict(cg=cg, branch=br.reshape(max_iter, P), rho=rt.reshape(max_iter, P),
                    gamma=gt.reshape(max_iter, P), r_feas=ft[: max_iter * p].reshape(max_iter, p),
                    r_evol=et)

    def get_support_log(self, max_iter):
        """per-iteration cardinality support fingerprints, (max_iter, p) uint64"""
        p = len(self.sets)
        out = np.zeros(max(1, max_iter * p), dtype=np.uint64)
        self._check(lib().sip_get_support_log(self.h, int(max_iter), _ptr(out)))
        return out[: max_iter * p].reshape(max_iter, p)

    def dykstra(self, m, x, max_outer=100, tol=1e-6, inner_max_iter=200, inner_tol=1e-3):
        """Algorithm 4 (parallel Dykstra, PARSDMM sub-problems): the Fig. 1
        comparator; returns the per-outer-iteration counters"""
        p = len(self.sets)
        b = dict(cg_max=np.zeros(max_outer, dtype=np.int32), l1_proj=np.zeros(max_outer, dtype=np.int32),
                 inner_iters=np.zeros(max_outer * p, dtype=np.int32), r_feas=np.zeros(max_outer * p),
                 r_evol=np.zeros(max_outer))
        lg = DykstraLog()
        lg.cg_max = b["cg_max"].ctypes.data_as(C.POINTER(C.c_int))
        lg.l1_proj = b["l1_proj"].ctypes.data_as(C.POINTER(C.c_int))
        lg.inner_iters = b["inner_iters"].ctypes.data_as(C.POINTER(C.c_int))
        lg.r_feas = b["r_feas"].ctypes.data_as(C.POINTER(C.c_double))
        lg.r_evol = b["r_evol"].ctypes.data_as(C.POINTER(C.c_double))
        s = self._check(lib().sip_dykstra(self.h, self._buf(m, self.N, "m"), self._buf(x, self.N, "x"),
                                          int(max_outer), float(tol), int(inner_max_iter), float(inner_tol),
                                          C.byref(lg)), (SIP_OK, SIP_NOT_CONVERGED))
        it = lg.iterations
        return dict(status=s, iterations=it, cg_max=b["cg_max"][:it].copy(), l1_proj=b["l1_proj"][:it].copy(),
                    inner_iters=b["inner_iters"].reshape(max_outer, p)[:it].copy(),
                    r_feas=b["r_feas"].reshape(max_outer, p)[:it].copy(), r_evol=b["r_evol"][:it].copy())

    def profile(self):
        """per-kernel-kind device ms and launch counts of the last project()"""
        n = len(KERNEL_KINDS)
        ms = np.zeros(n)
        cnt = np.zeros(n, dtype=np.int64)
        self._check(lib().sip_get_profile(self.h, n, _ptr(ms), _ptr(cnt)))
        return {k: (float(ms[i]), int(cnt[i])) for i, k in enumerate(KERNEL_KINDS)}

    def launch_count(self):
        n = C.c_int64(0)
        self._check(lib().sip_get_launch_count(self.h, C.byref(n)))
        return n.value


def _res(r, p):
    return dict(iterations=r.iterations, cg_iterations=r.cg_iterations, converged=bool(r.converged),
                breakdown=bool(r.breakdown), r_evol=r.r_evol, ms=r.ms,
                r_feas=np.array(r.r_feas[:p]), rho=np.array(r.rho[: p + 1]),
                gamma=np.array(r.gamma[: p + 1]))


def grid_for(problem, stream=None, comm=None):
    """Grid + sets for a sip_inputs.Problem (marshalling convenience); comm:
    a dist.comm_desc() for the z-slab path (the problem stays whole-grid)."""
    g = Grid(problem.shape, problem.h, problem.dtype, stream=stream, comm=comm)
    for sd in problem.sets:
        g.add_set(sd)
    return g


__all__ = ["Grid", "SipError", "lib", "grid_for", "EXPORTS"]
