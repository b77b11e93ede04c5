"""Seeded synthetic inputs for the PARSDMM hot path (BASELINE.json configs).

This module is shared by the oracle-side tests and the CUDA-side tests and
bench.  It holds NONE of the method's arithmetic: it draws the models m,
describes the constraint sets (as plain data) and computes problem
parameters that BASELINE.json defines in terms of the ground truth (C3's
TV radius and annulus radii, reading L4/L21).  Recipes: DESIGN.md section 4
(SURVEY.md 8(d)).  No item of the paper's datasets is reproduced; the
generators are stand-ins for the paper's seismic models (P:486-491,
P:526-531) and deblurring images.

Shapes are z-first: (nz, nx) in 2D, (nz, ny, nx) in 3D (reading L1).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

INF = float("inf")


@dataclass
class SetDef:
    """One constraint set V_i = {x : A_i x in C_i}, as data."""
    op: str                       # 'I','DZ','DY','DX','TV','BLUR_MASK'
    kind: str                     # 'bounds','l1','l2','annulus','card'
    lo: float = -INF
    hi: float = INF
    lo_vec: np.ndarray | None = None   # per-entry bounds, compact layout (length M)
    hi_vec: np.ndarray | None = None
    sigma: float = 0.0
    sigma_lo: float = 0.0
    sigma_hi: float = 0.0
    k: int = 0
    k_frac: float = 0.0
    relative: bool = False        # sigma*, k relative to A m (reading L4, L23)
    kernel: np.ndarray | None = None   # BLUR_MASK kernel (kh x kw)
    mask: np.ndarray | None = None     # BLUR_MASK observation mask, grid shape, uint8
    app_mode: str = ""            # '' whole vector, 'x' each row (x-fiber), 'z' each column


@dataclass
class Problem:
    name: str
    shape: tuple
    dtype: str                    # 'f32' or 'f64'
    m: np.ndarray                 # float64, grid shape
    sets: list
    h: tuple | None = None
    options: dict = field(default_factory=dict)
    n_levels: int = 1
    extra: dict = field(default_factory=dict)

    def __post_init__(self):
        # fp32 configurations: the model and per-entry bounds are the values
        # an fp32 run holds, so both sides of a parity test start from the
        # same bits (the oracle widens them exactly to fp64)
        if self.dtype == "f32":
            self.m = np.asarray(self.m, dtype=np.float64).astype(np.float32).astype(np.float64)
            for s in self.sets:
                for a in ("lo_vec", "hi_vec"):
                    v = getattr(s, a)
                    if v is not None:
                        setattr(s, a, np.asarray(v, dtype=np.float64).astype(np.float32).astype(np.float64))

    @property
    def N(self) -> int:
        return int(np.prod(self.shape))


DEFAULT_OPTIONS = dict(max_iter=200, n_cg=10, rho0=1e-2)   # BASELINE.json C1, reading L11


def gaussian_kernel(size=5, sigma=1.5):
    """normalised size x size Gaussian (reading L21)"""
    r = np.arange(size) - size // 2
    g = np.exp(-(r[:, None] ** 2 + r[None, :] ** 2) / (2.0 * sigma * sigma))
    return g / g.sum()


def _correlate_same(img, K):
    """'same' zero-padded correlation, used only to SYNTHESISE C3's data d"""
    kh, kw = K.shape
    pz, px = kh // 2, kw // 2
    pad = np.zeros((img.shape[0] + 2 * pz, img.shape[1] + 2 * px))
    pad[pz:pz + img.shape[0], px:px + img.shape[1]] = img
    out = np.zeros_like(img, dtype=np.float64)
    for a in range(kh):
        for b in range(kw):
            out += K[a, b] * pad[a:a + img.shape[0], b:b + img.shape[1]]
    return out


def _tv_l1(img):
    """||[D_z; (D_y;) D_x] img||_1 with h = 1 -- a problem PARAMETER (C3's
    radius is defined on the ground truth, which the solver never sees)"""
    return float(sum(np.abs(np.diff(img, axis=a)).sum() for a in range(img.ndim)))


# ----------------------------------------------------------------- C1
def c1_model(seed=0, shape=(64, 64)):
    rng = np.random.default_rng(seed)
    nz, nx = shape
    vel = rng.uniform(1500.0, 4500.0, size=10)          # draw order, unsorted
    layer = np.floor(10.0 * np.arange(nz) / nz).astype(int)
    m = np.repeat(vel[layer][:, None], nx, axis=1)
    m = m + rng.normal(0.0, 50.0, size=shape)
    return m


def c1(seed=0, shape=(64, 64)) -> Problem:
    m = c1_model(seed, shape)
    sets = [
        SetDef("I", "bounds", lo=1500.0, hi=4500.0),
        SetDef("TV", "l1", sigma=0.5, relative=True),
        SetDef("DZ", "bounds", lo=0.0, hi=1e4),
    ]
    return Problem("C1", shape, "f64", m, sets, options=dict(DEFAULT_OPTIONS))


# ----------------------------------------------------------------- C2
def c2_model(seed=1, shape=(512, 2048)):
    rng = np.random.default_rng(seed)
    nz, nx = shape
    depths = np.sort(rng.uniform(0.0, nz, size=11))
    dips = np.tan(np.deg2rad(rng.uniform(-8.0, 8.0, size=11)))
    vels = np.sort(rng.uniform(1500.0, 4200.0, size=12))
    zz = np.arange(nz, dtype=np.float64)[:, None]
    xx = np.arange(nx, dtype=np.float64)[None, :]
    m = np.full(shape, vels[0]) + 0.3 * zz
    for j in range(11):                       # layer j+1 below interface j
        top = depths[j] + dips[j] * (xx - nx / 2.0)
        below = zz >= top
        m = np.where(below, vels[j + 1] + 0.3 * (zz - top), m)
    for _ in range(3):                        # elliptical high-velocity bodies
        cz, cx = rng.uniform(0, nz), rng.uniform(0, nx)
        az, ax = rng.uniform(20, 80), rng.uniform(60, 250)
        th = rng.uniform(0, np.pi)
        dz, dx = zz - cz, xx - cx
        u = dz * np.cos(th) + dx * np.sin(th)
        v = -dz * np.sin(th) + dx * np.cos(th)
        m = np.where((u / az) ** 2 + (v / ax) ** 2 <= 1.0, 4700.0, m)
    m = np.clip(m, 1500.0, 4700.0)
    m = m + rng.normal(0.0, 100.0, size=shape)
    return m


def c2(seed=1, shape=(512, 2048)) -> Problem:
    m = c2_model(seed, shape)
    sets = [
        SetDef("I", "bounds", lo=1500.0, hi=4700.0),
        SetDef("TV", "l1", sigma=0.3, relative=True),
        SetDef("DX", "card", k_frac=0.05, relative=True),
        SetDef("DZ", "bounds", lo=0.0, hi=INF),
    ]
    return Problem("C2", shape, "f32", m, sets, options=dict(DEFAULT_OPTIONS))


# ----------------------------------------------------------------- C3
def c3_data(seed=2, shape=(1024, 1024)):
    rng = np.random.default_rng(seed)
    nz, nx = shape
    truth = np.full(shape, rng.uniform(0.0, 255.0))
    zz = np.arange(nz)[:, None]
    xx = np.arange(nx)[None, :]
    scale = min(nz, nx) / 1024.0
    for _ in range(40):
        val = rng.uniform(0.0, 255.0)
        if rng.uniform() < 0.5:
            hz, hx = rng.uniform(32, 256) * scale, rng.uniform(32, 256) * scale
            z0, x0 = rng.uniform(0, nz), rng.uniform(0, nx)
            sel = (zz >= z0) & (zz < z0 + hz) & (xx >= x0) & (xx < x0 + hx)
        else:
            r = rng.uniform(16, 128) * scale
            z0, x0 = rng.uniform(0, nz), rng.uniform(0, nx)
            sel = (zz - z0) ** 2 + (xx - x0) ** 2 <= r * r
        truth = np.where(sel, val, truth)
    K = gaussian_kernel(5, 1.5)
    mask = (rng.uniform(size=shape) < 0.5).astype(np.uint8)
    blurred = _correlate_same(truth, K)
    d = np.where(mask == 1, blurred + rng.normal(0.0, 8.0, size=shape), 0.0)
    return truth, K, mask, d


def c3(seed=2, shape=(1024, 1024)) -> Problem:
    truth, K, mask, d = c3_data(seed, shape)
    kept = mask.ravel() == 1
    dk = d.ravel()[kept]
    m = np.where(mask == 1, d, dk.mean())              # reading L22
    tnorm = float(np.sqrt((truth ** 2).sum()))
    sets = [
        SetDef("BLUR_MASK", "bounds", lo_vec=dk - 16.0, hi_vec=dk + 16.0, kernel=K, mask=mask),
        SetDef("I", "bounds", lo=0.0, hi=255.0),
        SetDef("TV", "l1", sigma=0.2 * _tv_l1(truth)),
        SetDef("I", "annulus", sigma_lo=0.9 * tnorm, sigma_hi=1.1 * tnorm),
    ]
    return Problem("C3", shape, "f32", m, sets, options=dict(DEFAULT_OPTIONS),
                   extra=dict(truth=truth, d=d))


# ----------------------------------------------------------------- C4 / C5
def c45_model(seed, shape):
    rng = np.random.default_rng(seed)
    nz, ny, nx = shape
    vels = np.sort(rng.uniform(1500.0, 4000.0, size=10))
    layer = np.floor(10.0 * np.arange(nz) / nz).astype(int)
    m = np.empty(shape, dtype=np.float64)
    m[:] = vels[layer][:, None, None]
    for _ in range(5):                         # separable Gaussian anomalies
        c = [rng.uniform(0, n) for n in shape]
        s = [rng.uniform(5, 25) for _ in range(3)]
        a = rng.uniform(-500.0, 500.0)
        gz = np.exp(-((np.arange(nz) - c[0]) ** 2) / (2 * s[0] ** 2))
        gy = np.exp(-((np.arange(ny) - c[1]) ** 2) / (2 * s[1] ** 2))
        gx = np.exp(-((np.arange(nx) - c[2]) ** 2) / (2 * s[2] ** 2))
        m += a * gz[:, None, None] * gy[None, :, None] * gx[None, None, :]
    m += rng.normal(0.0, 50.0, size=shape)
    return m


def c4(seed=3, shape=(256, 256, 128)) -> Problem:
    m = c45_model(seed, shape)
    sets = [
        SetDef("I", "bounds", lo=1500.0, hi=4500.0),
        SetDef("TV", "l1", sigma=0.3, relative=True),
        SetDef("DZ", "bounds", lo=0.0, hi=INF),
    ]
    return Problem("C4", shape, "f32", m, sets, options=dict(DEFAULT_OPTIONS))


def c5(seed=4, shape=(512, 512, 256)) -> Problem:
    m = c45_model(seed, shape)
    sets = [
        SetDef("I", "bounds", lo=1500.0, hi=4500.0),
        SetDef("TV", "l1", sigma=0.3, relative=True),
        SetDef("DZ", "bounds", lo=0.0, hi=INF),
        SetDef("DZ", "card", k_frac=0.02, relative=True),
        SetDef("I", "annulus", sigma_lo=0.95, sigma_hi=1.05, relative=True),
    ]
    return Problem("C5", shape, "f32", m, sets, options=dict(DEFAULT_OPTIONS), n_levels=3)


CONFIGS = {"C1": c1, "C2": c2, "C3": c3, "C4": c4, "C5": c5}


# ----------------------------------------------------------------- tiny (T3)
def tiny_model(seed, shape):
    """layered model + noise, the C1/C4 recipe at small size"""
    rng = np.random.default_rng(seed)
    nz = shape[0]
    nl = max(2, min(5, nz // 2))
    vel = rng.uniform(1500.0, 4500.0, size=nl)
    layer = np.floor(nl * np.arange(nz) / nz).astype(int)
    m = np.broadcast_to(vel[layer].reshape((nz,) + (1,) * (len(shape) - 1)), shape).copy()
    return m + rng.normal(0.0, 150.0, size=shape)


def tiny(seed=100, shape=(8, 8), kinds=("bounds", "l1", "slope")) -> Problem:
    """tiny parity case: every set type available by name"""
    m = tiny_model(seed, shape)
    sets = []
    for k in kinds:
        if k == "bounds":
            sets.append(SetDef("I", "bounds", lo=1500.0, hi=4500.0))
        elif k == "l1":
            sets.append(SetDef("TV", "l1", sigma=0.5, relative=True))
        elif k == "slope":
            sets.append(SetDef("DZ", "bounds", lo=0.0, hi=INF))
        elif k == "dxbox":
            sets.append(SetDef("DX", "bounds", lo=-200.0, hi=200.0))
        elif k == "dybox":
            sets.append(SetDef("DY", "bounds", lo=-200.0, hi=200.0))
        elif k == "card":
            sets.append(SetDef("DX", "card", k_frac=0.25, relative=True))
        elif k == "cardz":
            sets.append(SetDef("DZ", "card", k_frac=0.2, relative=True))
        elif k == "annulus":
            sets.append(SetDef("I", "annulus", sigma_lo=0.95, sigma_hi=0.99, relative=True))
        elif k == "l2":
            sets.append(SetDef("DZ", "l2", sigma=0.5, relative=True))
        elif k == "l1x":
            sets.append(SetDef("DX", "l1", sigma=0.4, relative=True))
        # per-fiber sets (NEXT-1): x-fibers are rows, z-fibers columns
        elif k == "card_rows":
            sets.append(SetDef("DX", "card", k_frac=0.3, relative=True, app_mode="x"))
        elif k == "card_cols":
            sets.append(SetDef("DZ", "card", k_frac=0.3, relative=True, app_mode="z"))
        elif k == "l1_rows":
            sets.append(SetDef("DX", "l1", sigma=120.0 * (shape[-1] - 1), app_mode="x"))
        elif k == "l1_cols":
            sets.append(SetDef("I", "l1", sigma=2500.0 * shape[0], app_mode="z"))
        elif k == "l2_rows":
            sets.append(SetDef("DX", "l2", sigma=150.0 * np.sqrt(shape[-1] - 1), app_mode="x"))
        elif k == "ann_cols":
            sets.append(SetDef("I", "annulus", sigma_lo=2400.0 * np.sqrt(shape[0]),
                               sigma_hi=3200.0 * np.sqrt(shape[0]), app_mode="z"))
        else:
            raise KeyError(k)
    return Problem(f"tiny{seed}", tuple(shape), "f64", m, sets,
                   options=dict(DEFAULT_OPTIONS))


def tiny_blur(seed=150, shape=(12, 10)) -> Problem:
    """tiny C3-like case (blur+mask data constraint), fp64"""
    truth, K, mask, d = c3_data(seed, shape)
    kept = mask.ravel() == 1
    dk = d.ravel()[kept]
    m = np.where(mask == 1, d, dk.mean())
    tnorm = float(np.sqrt((truth ** 2).sum()))
    sets = [
        SetDef("BLUR_MASK", "bounds", lo_vec=dk - 16.0, hi_vec=dk + 16.0, kernel=K, mask=mask),
        SetDef("I", "bounds", lo=0.0, hi=255.0),
        SetDef("TV", "l1", sigma=0.2 * _tv_l1(truth)),
        SetDef("I", "annulus", sigma_lo=0.9 * tnorm, sigma_hi=1.1 * tnorm),
    ]
    return Problem(f"tinyblur{seed}", tuple(shape), "f64", m, sets,
                   options=dict(DEFAULT_OPTIONS), extra=dict(truth=truth, d=d))
