"""CPU ORACLE for PARSDMM (arXiv 1902.09699) -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import this package.  The
product path (``paper_1902_09699_b200``) never imports it and shares no
code with it.  This module is ctypes marshalling over ``sipref.c`` (plain
C99, fp64, single-threaded); all arithmetic of the method lives in that C
file, each function citing the passage of PAPER.md it follows.

Layouts are the paper's compact ones (see ``sipref.h``).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sipref.c")
_LIB = os.path.join(_HERE, "libsipref.so")

OPS = {"I": 0, "DZ": 1, "DY": 2, "DX": 3, "TV": 4, "BLUR_MASK": 5}
KINDS = {"bounds": 0, "l1": 1, "l2": 2, "annulus": 3, "card": 4, "rank": 5, "nuclear": 6, "dct_l1": 7, "haar_l1": 8}
BRANCH = {0: "both", 1: "alpha", 2: "beta", 3: "none", -1: "-"}


def build(force: bool = False) -> str:
    """Compile sipref.c with gcc (-O2 -ffp-contract=off, no OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "sipref.h"))
    ):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-std=c99", "-O2", "-ffp-contract=off", "-fPIC", "-shared",
             "-Wall", "-o", tmp, _SRC, "-lm"]
        )
        os.replace(tmp, _LIB)
    return _LIB


class Grid(C.Structure):
    _fields_ = [("ndim", C.c_int), ("n", C.c_int64 * 3), ("h", C.c_double * 3)]


class Set(C.Structure):
    _fields_ = [
        ("op", C.c_int), ("type", C.c_int),
        ("lo", C.c_double), ("hi", C.c_double),
        ("lo_vec", C.POINTER(C.c_double)), ("hi_vec", C.POINTER(C.c_double)),
        ("sigma", C.c_double), ("sigma_lo", C.c_double), ("sigma_hi", C.c_double),
        ("k", C.c_int64), ("relative", C.c_int), ("k_frac", C.c_double),
        ("kernel", C.POINTER(C.c_double)), ("kh", C.c_int), ("kw", C.c_int),
        ("mask", C.POINTER(C.c_ubyte)),
        ("app_mode", C.c_int), ("fib_len", C.c_int64),
        ("tgrid", Grid), ("mrows", C.c_int64), ("mcols", C.c_int64),
    ]


class Options(C.Structure):
    _fields_ = [
        ("max_iter", C.c_int), ("n_cg", C.c_int),
        ("rho0", C.c_double), ("gamma0", C.c_double), ("eps_evol", C.c_double),
        ("eps_feas", C.c_double), ("eps_corr", C.c_double),
        ("adapt_every", C.c_int), ("check_every", C.c_int), ("hist_s", C.c_int),
        ("rho_ratio_cap", C.c_double), ("gamma_max", C.c_double),
        ("eq25", C.c_int), ("fixed_work", C.c_int), ("cg_tol_floor", C.c_double),
    ]


class Log(C.Structure):
    _fields_ = [
        ("iterations", C.c_int), ("cg_total", C.c_int), ("converged", C.c_int),
        ("breakdown", C.c_int), ("r_evol", C.c_double),
        ("cg_per_iter", C.POINTER(C.c_int)), ("branch", C.POINTER(C.c_int)),
        ("rho_trace", C.POINTER(C.c_double)), ("gamma_trace", C.POINTER(C.c_double)),
        ("r_feas_trace", C.POINTER(C.c_double)), ("r_evol_trace", C.POINTER(C.c_double)),
        ("supp_hash", C.POINTER(C.c_uint64)),
        ("r_feas", C.POINTER(C.c_double)), ("rho", C.POINTER(C.c_double)),
        ("gamma", C.POINTER(C.c_double)),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _lib.sipref_npts.restype = C.c_int64
        _lib.sipref_op_len.restype = C.c_int64
        _lib.sipref_fiber_len.restype = C.c_int64
        _lib.sipref_feas.restype = C.c_double
        _lib.sipref_supp_key.restype = C.c_uint64
        _lib.sipref_supp_key.argtypes = [C.POINTER(Grid), C.c_int, C.c_int64]
    return _lib


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _ip(a):
    return a.ctypes.data_as(C.POINTER(C.c_int))


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def make_grid(shape, h=None) -> Grid:
    """shape is z-first: (nz, nx) or (nz, ny, nx)."""
    g = Grid()
    if len(shape) == 2:
        g.ndim = 2
        g.n[:] = [shape[0], 1, shape[1]]
        hh = h or (1.0, 1.0)
        g.h[:] = [hh[0], 1.0, hh[1]]
    else:
        g.ndim = 3
        g.n[:] = list(shape)
        hh = h or (1.0, 1.0, 1.0)
        g.h[:] = list(hh)
    return g


class _SetHolder:
    """keeps numpy buffers referenced by a ctypes Set alive"""

    def __init__(self, sd):
        self.keep = []
        s = Set()
        s.op = OPS[sd.op]
        s.type = KINDS[sd.kind]
        s.lo, s.hi = float(sd.lo), float(sd.hi)
        if sd.lo_vec is not None:
            a = _f64(sd.lo_vec).ravel(); self.keep.append(a); s.lo_vec = _dp(a)
        if sd.hi_vec is not None:
            a = _f64(sd.hi_vec).ravel(); self.keep.append(a); s.hi_vec = _dp(a)
        s.sigma = float(sd.sigma)
        s.sigma_lo, s.sigma_hi = float(sd.sigma_lo), float(sd.sigma_hi)
        s.k = int(sd.k)
        s.relative = int(bool(sd.relative))
        s.k_frac = float(sd.k_frac)
        s.app_mode = APP_MODES[getattr(sd, "app_mode", "") or ""]
        if sd.kernel is not None:
            kk = _f64(sd.kernel); self.keep.append(kk)
            s.kernel = _dp(kk); s.kh, s.kw = kk.shape
        if sd.mask is not None:
            mm = np.ascontiguousarray(sd.mask, dtype=np.uint8).ravel(); self.keep.append(mm)
            s.mask = mm.ctypes.data_as(C.POINTER(C.c_ubyte))
        self.s = s


def _sets_array(setdefs):
    holders = [_SetHolder(sd) for sd in setdefs]
    arr = (Set * max(1, len(holders)))()
    for i, h in enumerate(holders):
        arr[i] = h.s
    return arr, holders


def options(**kw) -> Options:
    o = Options()
    lib().sipref_default_options(C.byref(o))
    for k, v in kw.items():
        if not hasattr(o, k):
            raise KeyError(k)
        setattr(o, k, v)
    return o


# ---------------------------------------------------------------- operators
def op_len(shape, sd, h=None) -> int:
    g = make_grid(shape, h)
    hold = _SetHolder(sd)
    return int(lib().sipref_op_len(C.byref(g), C.byref(hold.s)))


def apply_A(shape, sd, x, h=None):
    g = make_grid(shape, h)
    hold = _SetHolder(sd)
    M = int(lib().sipref_op_len(C.byref(g), C.byref(hold.s)))
    x = _f64(x).ravel()
    y = np.zeros(M)
    lib().sipref_apply_A(C.byref(g), C.byref(hold.s), _dp(x), _dp(y))
    return y


def apply_AT(shape, sd, y, h=None):
    g = make_grid(shape, h)
    hold = _SetHolder(sd)
    y = _f64(y).ravel()
    x = np.zeros(int(np.prod(shape)))
    lib().sipref_apply_AT(C.byref(g), C.byref(hold.s), _dp(y), _dp(x))
    return x


def apply_C(shape, setdefs, rho, p_vec, h=None):
    g = make_grid(shape, h)
    arr, _hold = _sets_array(setdefs)
    rho = _f64(rho)
    pv = _f64(p_vec).ravel()
    q = np.zeros_like(pv)
    lib().sipref_apply_C(C.byref(g), len(setdefs), arr, _dp(rho), _dp(pv), _dp(q))
    return q


APP_MODES = {"": 0, "x": 1, "z": 2}


def fiber_len(shape, sd, h=None) -> int:
    g = make_grid(shape, h)
    hold = _SetHolder(sd)
    return int(lib().sipref_fiber_len(C.byref(g), C.byref(hold.s)))


def matrix_shape(shape, op):
    """(rows, cols) of one matrix of the view of op's output (reading L29)"""
    g = make_grid(shape)
    r, c = C.c_int64(0), C.c_int64(0)
    lib().sipref_matrix_shape(C.byref(g), OPS[op], C.byref(r), C.byref(c))
    return r.value, c.value


def dct(shape, x, inverse=False):
    """orthonormal DCT-II along every axis of a grid field (or its inverse)"""
    g = make_grid(shape)
    x = _f64(x).ravel()
    y = np.zeros_like(x)
    lib().sipref_dct(C.byref(g), int(bool(inverse)), _dp(x), _dp(y))
    return y


def haar(shape, x, inverse=False):
    """orthonormal full-depth Haar transform along every axis (or its inverse)"""
    g = make_grid(shape)
    x = _f64(x).ravel()
    y = np.zeros_like(x)
    lib().sipref_haar(C.byref(g), int(bool(inverse)), _dp(x), _dp(y))
    return y


def svd_values(a):
    """singular values of a 2D array (one-sided Jacobi, descending)"""
    a = _f64(a)
    r, c = a.shape
    sv = np.zeros(min(r, c))
    lib().sipref_svd_values(C.c_int64(r), C.c_int64(c), _dp(a.ravel()), _dp(sv))
    return sv


def project(sd, w, shape=None):
    """Table 1 projector; shape is needed for per-fiber sets (app_mode) and
    the matrix view of rank / nuclear-norm sets"""
    hold = _SetHolder(sd)
    if shape is not None:
        hold.s.fib_len = fiber_len(shape, sd)
        hold.s.mrows, hold.s.mcols = matrix_shape(shape, sd.op)
        hold.s.tgrid = make_grid(shape)
    w = _f64(w).ravel()
    y = np.zeros_like(w)
    lib().sipref_project(C.byref(hold.s), C.c_int64(w.size), _dp(w), _dp(y))
    return y


def prox_dist(m, rho, w):
    m = _f64(m).ravel(); w = _f64(w).ravel()
    y = np.zeros_like(w)
    lib().sipref_prox_dist(C.c_int64(w.size), _dp(m), C.c_double(rho), _dp(w), _dp(y))
    return y


def feas(sd, s_vec, shape=None):
    hold = _SetHolder(sd)
    if shape is not None:
        hold.s.fib_len = fiber_len(shape, sd)
        hold.s.mrows, hold.s.mcols = matrix_shape(shape, sd.op)
        hold.s.tgrid = make_grid(shape)
    s_vec = _f64(s_vec).ravel()
    return float(lib().sipref_feas(C.byref(hold.s), C.c_int64(s_vec.size), _dp(s_vec)))


def cg(shape, setdefs, rho, b, x0, n_cg, eq25=True, h=None):
    g = make_grid(shape, h)
    arr, _hold = _sets_array(setdefs)
    rho = _f64(rho); b = _f64(b).ravel(); x = _f64(x0).ravel().copy()
    tol = C.c_double(0); bd = C.c_int(0)
    it = lib().sipref_cg(C.byref(g), len(setdefs), arr, _dp(rho), _dp(b), _dp(x),
                         int(n_cg), int(eq25), C.byref(tol), C.byref(bd))
    return x, int(it), float(tol.value), int(bd.value)


def adapt_rho_gamma(v_hat, v_hat0, v, v0, s, s0, y, y0, rho, eps_corr=0.3):
    arrs = [_f64(a).ravel() for a in (v_hat, v_hat0, v, v0, s, s0, y, y0)]
    rn = C.c_double(0); gn = C.c_double(0)
    br = lib().sipref_adapt_rho_gamma(C.c_int64(arrs[0].size), *[_dp(a) for a in arrs],
                                      C.c_double(rho), C.c_double(eps_corr),
                                      C.byref(rn), C.byref(gn))
    return float(rn.value), float(gn.value), int(br)


# ---------------------------------------------------------------- PARSDMM
@dataclass
class Result:
    x: np.ndarray
    status: int
    iterations: int
    cg_total: int
    converged: bool
    breakdown: bool
    r_evol: float
    r_feas: np.ndarray
    rho: np.ndarray
    gamma: np.ndarray
    cg_per_iter: np.ndarray
    branch: np.ndarray
    rho_trace: np.ndarray
    gamma_trace: np.ndarray
    r_feas_trace: np.ndarray
    r_evol_trace: np.ndarray
    supp_hash: np.ndarray = None
    y: list = field(default_factory=list)
    v: list = field(default_factory=list)


def _make_log(p, max_iter):
    P = p + 1
    bufs = dict(
        cg_per_iter=np.zeros(max_iter, dtype=np.int32),
        branch=np.full(max_iter * P, -1, dtype=np.int32),
        rho_trace=np.zeros(max_iter * P), gamma_trace=np.zeros(max_iter * P),
        r_feas_trace=np.full(max(1, max_iter * p), np.nan),
        r_evol_trace=np.full(max_iter, np.nan),
        supp_hash=np.zeros(max(1, max_iter * p), dtype=np.uint64),
        r_feas=np.zeros(max(1, p)), rho=np.zeros(P), gamma=np.zeros(P),
    )
    lg = Log()
    lg.cg_per_iter = _ip(bufs["cg_per_iter"]); lg.branch = _ip(bufs["branch"])
    lg.supp_hash = bufs["supp_hash"].ctypes.data_as(C.POINTER(C.c_uint64))
    for k in ("rho_trace", "gamma_trace", "r_feas_trace", "r_evol_trace", "r_feas", "rho", "gamma"):
        setattr(lg, k, _dp(bufs[k]))
    return lg, bufs


def _result(x, st, lg, bufs, p, max_iter, ys=None, vs=None):
    P = p + 1
    it = lg.iterations
    return Result(
        x=x, status=int(st), iterations=int(it), cg_total=int(lg.cg_total),
        converged=bool(lg.converged), breakdown=bool(lg.breakdown), r_evol=float(lg.r_evol),
        r_feas=bufs["r_feas"][:p].copy(), rho=bufs["rho"].copy(), gamma=bufs["gamma"].copy(),
        cg_per_iter=bufs["cg_per_iter"][:it].copy(),
        branch=bufs["branch"].reshape(max_iter, P)[:it].copy(),
        rho_trace=bufs["rho_trace"].reshape(max_iter, P)[:it].copy(),
        gamma_trace=bufs["gamma_trace"].reshape(max_iter, P)[:it].copy(),
        r_feas_trace=bufs["r_feas_trace"][: max_iter * p].reshape(max_iter, p)[:it].copy()
        if p else np.zeros((it, 0)),
        r_evol_trace=bufs["r_evol_trace"][:it].copy(),
        supp_hash=bufs["supp_hash"][: max_iter * p].reshape(max_iter, p)[:it].copy()
        if p else np.zeros((it, 0), dtype=np.uint64),
        y=ys or [], v=vs or [],
    )


def parsdmm(shape, setdefs, m, h=None, want_yv=False, init=None, **opts):
    """Algorithm 1.  init: optional dict(x=..., y=[...], v=[...], rho=..., gamma=...)."""
    g = make_grid(shape, h)
    arr, _hold = _sets_array(setdefs)
    o = options(**opts)
    p = len(setdefs)
    m = _f64(m).ravel()
    N = m.size
    x = np.zeros(N)
    lg, bufs = _make_log(p, o.max_iter)
    Ms = [op_len(shape, sd, h) for sd in setdefs] + [N]
    keep = []

    def ptr_array(vecs):
        a = (C.POINTER(C.c_double) * (p + 1))()
        for i, v in enumerate(vecs):
            keep.append(v)
            a[i] = _dp(v)
        return a

    ix = iy = iv = ir = ig = None
    if init is not None:
        if init.get("x") is not None:
            ix = _f64(init["x"]).ravel(); keep.append(ix); ix = _dp(ix)
        if init.get("y") is not None:
            iy = ptr_array([_f64(a).ravel().copy() for a in init["y"]])
        if init.get("v") is not None:
            iv = ptr_array([_f64(a).ravel().copy() for a in init["v"]])
        if init.get("rho") is not None:
            r = _f64(init["rho"]); keep.append(r); ir = _dp(r)
        if init.get("gamma") is not None:
            gg = _f64(init["gamma"]); keep.append(gg); ig = _dp(gg)
    ys = vs = None
    oy = ov = None
    if want_yv:
        ys = [np.zeros(Mi) for Mi in Ms]
        vs = [np.zeros(Mi) for Mi in Ms]
        oy = ptr_array(ys); ov = ptr_array(vs)
    st = lib().sipref_parsdmm(C.byref(g), p, arr, C.byref(o), _dp(m), _dp(x), ix, iy, iv,
                              ir, ig, oy, ov, C.byref(lg))
    return _result(x, st, lg, bufs, p, o.max_iter, ys, vs)


def parsdmm_multilevel(shape, setdefs, m, n_levels, h=None, **opts):
    g = make_grid(shape, h)
    arr, _hold = _sets_array(setdefs)
    o = options(**opts)
    p = len(setdefs)
    m = _f64(m).ravel()
    x = np.zeros(m.size)
    logs = (Log * n_levels)()
    allbufs = []
    for l in range(n_levels):
        lg, bufs = _make_log(p, o.max_iter)
        logs[l] = lg
        allbufs.append(bufs)
    st = lib().sipref_parsdmm_multilevel(C.byref(g), p, arr, C.byref(o), int(n_levels),
                                         _dp(m), _dp(x), logs)
    if st < 0:
        raise ValueError(f"sipref_parsdmm_multilevel: error {st}")
    return x, st, [_result(None, st, logs[l], allbufs[l], p, o.max_iter) for l in range(n_levels)]


class DykLog(C.Structure):
    _fields_ = [("iterations", C.c_int), ("cg_max", C.POINTER(C.c_int)), ("l1_proj", C.POINTER(C.c_int)),
                ("inner_iters", C.POINTER(C.c_int)), ("r_feas", C.POINTER(C.c_double)),
                ("r_evol", C.POINTER(C.c_double))]


def dykstra(shape, setdefs, m, max_outer=100, tol=1e-6, h=None, **inner_opts):
    """Algorithm 4 with PARSDMM sub-problems (the Fig. 1 comparator)"""
    g = make_grid(shape, h)
    arr, _hold = _sets_array(setdefs)
    o = options(**inner_opts)
    p = len(setdefs)
    m = _f64(m).ravel()
    x = np.zeros(m.size)
    b = dict(cg_max=np.zeros(max_outer, dtype=np.int32), l1_proj=np.zeros(max_outer, dtype=np.int32),
             inner_iters=np.zeros(max_outer * p, dtype=np.int32), r_feas=np.zeros(max_outer * p),
             r_evol=np.zeros(max_outer))
    lg = DykLog()
    lg.cg_max = _ip(b["cg_max"]); lg.l1_proj = _ip(b["l1_proj"]); lg.inner_iters = _ip(b["inner_iters"])
    lg.r_feas = _dp(b["r_feas"]); lg.r_evol = _dp(b["r_evol"])
    st = lib().sipref_dykstra(C.byref(g), p, arr, C.byref(o), int(max_outer), C.c_double(tol), _dp(m),
                              _dp(x), C.byref(lg))
    it = lg.iterations
    return dict(x=x, status=int(st), iterations=it, cg_max=b["cg_max"][:it].copy(),
                l1_proj=b["l1_proj"][:it].copy(), inner_iters=b["inner_iters"].reshape(max_outer, p)[:it].copy(),
                r_feas=b["r_feas"].reshape(max_outer, p)[:it].copy(), r_evol=b["r_evol"][:it].copy())


def restrict(shape, f):
    g = make_grid(shape)
    f = _f64(f).ravel()
    cshape = tuple(s // 2 for s in shape)
    c = np.zeros(int(np.prod(cshape)))
    lib().sipref_restrict(C.byref(g), _dp(f), _dp(c))
    return c.reshape(cshape)


def prolong_field(cshape, fshape, op, c):
    """sipref_prolong_field: the coarse field of operator op (compact) on the
    fine grid (compact)"""
    cg, fg = make_grid(cshape), make_grid(fshape)
    c = _f64(c).ravel()
    from sip_inputs import SetDef  # plain data holder
    M = op_len(fshape, SetDef(op, "bounds"))
    f = np.zeros(M)
    lib().sipref_prolong_field(C.byref(cg), C.byref(fg), OPS[op], _dp(c), _dp(f))
    return f


def resolve_set(shape, sd, m, h=None):
    """sipref_resolve_set: (sigma, sigma_lo, sigma_hi, k) of a relative set"""
    g = make_grid(shape, h)
    hold = _SetHolder(sd)
    out = Set()
    m = _f64(m).ravel()
    lib().sipref_resolve_set(C.byref(g), C.byref(hold.s), _dp(m), C.byref(out))
    return float(out.sigma), float(out.sigma_lo), float(out.sigma_hi), int(out.k)


def interp(c, fshape):
    c = _f64(c)
    cs = c.shape if c.ndim == 3 else (c.shape[0], 1, c.shape[1])
    fs = fshape if len(fshape) == 3 else (fshape[0], 1, fshape[1])
    f = np.zeros(int(np.prod(fs)))
    lib().sipref_interp(C.c_int64(cs[0]), C.c_int64(cs[1]), C.c_int64(cs[2]), _dp(c.ravel()),
                        C.c_int64(fs[0]), C.c_int64(fs[1]), C.c_int64(fs[2]), _dp(f))
    return f.reshape(fshape)


def supp_key(shape, op, j, h=None) -> int:
    """support fingerprint key of compact entry j of operator op's output"""
    g = make_grid(shape, h)
    return int(lib().sipref_supp_key(C.byref(g), OPS[op], int(j)))


def supp_hash(shape, op, y, h=None) -> int:
    """sum (mod 2^64) of the keys of the non-zero entries of y (compact)"""
    s = 0
    for j in np.flatnonzero(np.asarray(y).ravel() != 0.0):
        s = (s + supp_key(shape, op, int(j), h)) & 0xFFFFFFFFFFFFFFFF
    return s


def relres(a, b):
    """relative L2 difference ||a-b||/||b|| (b the reference)"""
    a = np.asarray(a, dtype=np.float64).ravel(); b = np.asarray(b, dtype=np.float64).ravel()
    nb = float(np.linalg.norm(b))
    return float(np.linalg.norm(a - b)) / (nb if nb > 0 else 1.0)

