"""Pins of the CPU oracle against what the paper and mathematics fix.

CPU-only (runs under ``-m "not gpu"``).  Each test pins one oracle function
to something other than the oracle itself: worked examples (tests/golden,
each cited), closed forms, invariants, brute force on tiny inputs, textbook
or library routines (numpy.linalg.solve, scipy isotonic regression, scipy
SLSQP) and Dykstra's algorithm (paper Algorithm 4).
"""
import itertools
import json
import os

import numpy as np
import pytest
import scipy.optimize as so

import oracle as O
from sip_inputs import INF, SetDef, gaussian_kernel, tiny_model

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))
rng0 = np.random.default_rng(12345)


def dense_of(shape, sd, h=None):
    """dense matrix of an oracle operator, column by column (A e_j)"""
    N = int(np.prod(shape))
    cols = [O.apply_A(shape, sd, np.eye(N)[j], h) for j in range(N)]
    return np.stack(cols, axis=1)


def dense_T(shape, sd, M, h=None):
    rows = [O.apply_AT(shape, sd, np.eye(M)[j], h) for j in range(M)]
    return np.stack(rows, axis=0)   # row j = A^T e_j  ->  equals A


def d1(n, h=1.0):
    """Eq. 8: (n-1) x n bidiagonal (-1, 1)/h"""
    D = np.zeros((n - 1, n))
    for i in range(n - 1):
        D[i, i], D[i, i + 1] = -1.0, 1.0
    return D / h


# ------------------------------------------------------------ operators
def test_dz_worked_example():
    g = GOLD["dz_2x2"]
    A = dense_of(tuple(g["shape"]), SetDef("DZ", "bounds"))
    np.testing.assert_array_equal(A, np.array(g["matrix"], dtype=float))


@pytest.mark.parametrize("shape,h", [((5, 4), (2.0, 3.0)), ((3, 4, 5), (2.0, 0.5, 3.0))])
def test_operators_kronecker(shape, h):
    """the 2D vertical derivative is D_z (x) I_x; lateral ones I (x) D."""
    if len(shape) == 2:
        nz, nx = shape
        Dz = np.kron(d1(nz, h[0]), np.eye(nx))
        Dx = np.kron(np.eye(nz), d1(nx, h[1]))
        blocks = [Dz, Dx]
        ops = [("DZ", Dz), ("DX", Dx)]
    else:
        nz, ny, nx = shape
        Dz = np.kron(d1(nz, h[0]), np.eye(ny * nx))
        Dy = np.kron(np.eye(nz), np.kron(d1(ny, h[1]), np.eye(nx)))
        Dx = np.kron(np.eye(nz * ny), d1(nx, h[2]))
        blocks = [Dz, Dy, Dx]
        ops = [("DZ", Dz), ("DY", Dy), ("DX", Dx)]
    for op, ref in ops:
        np.testing.assert_allclose(dense_of(shape, SetDef(op, "bounds"), h), ref, atol=1e-15)
    np.testing.assert_allclose(dense_of(shape, SetDef("TV", "l1"), h), np.vstack(blocks), atol=1e-15)
    N = int(np.prod(shape))
    np.testing.assert_array_equal(dense_of(shape, SetDef("I", "bounds"), h), np.eye(N))


@pytest.mark.parametrize("shape", [(6, 7), (4, 5, 6)])
def test_operators_constants_and_ramps(shape):
    """derivatives annihilate constants; a unit-slope ramp maps to 1"""
    h = (2.0, 0.5) if len(shape) == 2 else (2.0, 0.25, 0.5)
    c = np.full(shape, 3.7)
    for op in (["DZ", "DX"] if len(shape) == 2 else ["DZ", "DY", "DX"]):
        assert np.abs(O.apply_A(shape, SetDef(op, "bounds"), c, h)).max() == 0.0
    axes = {"DZ": 0, "DY": 1, "DX": len(shape) - 1}
    for op, ax in axes.items():
        if op == "DY" and len(shape) == 2:
            continue
        idx = np.indices(shape)[ax].astype(float) * h[ax]
        np.testing.assert_allclose(O.apply_A(shape, SetDef(op, "bounds"), idx, h), 1.0, rtol=1e-14)


def _blur_set(shape, seed=0, sym=False):
    r = np.random.default_rng(seed)
    K = gaussian_kernel(5, 1.5) if sym else r.uniform(0.1, 1.0, size=(3, 5))
    mask = (r.uniform(size=shape) < 0.6).astype(np.uint8)
    return SetDef("BLUR_MASK", "bounds", kernel=K, mask=mask)


@pytest.mark.parametrize("shape", [(7, 9), (4, 5, 6), (9, 6)])
def test_adjoint_identity(shape):
    """<A a, b> = <a, A^T b> within 1e-12 for every operator"""
    ops = ["I", "DZ", "DX", "TV"] + (["DY"] if len(shape) == 3 else ["BLUR"])
    r = np.random.default_rng(7)
    for op in ops:
        sd = _blur_set(shape) if op == "BLUR" else SetDef(op, "bounds")
        M = O.op_len(shape, sd)
        for _ in range(5):
            a = r.normal(size=int(np.prod(shape)))
            b = r.normal(size=M)
            lhs = O.apply_A(shape, sd, a) @ b
            rhs = a @ O.apply_AT(shape, sd, b)
            assert abs(lhs - rhs) <= 1e-12 * np.linalg.norm(a) * np.linalg.norm(b) * 10


def test_blur_delta_response():
    """G is a 'same' correlation (reading L21): a delta returns the mirrored
    kernel; the restriction S keeps the masked pixels in index order"""
    shape = (9, 11)
    K = np.arange(15, dtype=float).reshape(3, 5) + 1.0
    x = np.zeros(shape); x[4, 5] = 1.0
    full = SetDef("BLUR_MASK", "bounds", kernel=K, mask=np.ones(shape, np.uint8))
    y = O.apply_A(shape, full, x).reshape(shape)
    np.testing.assert_array_equal(y[3:6, 3:8], K[::-1, ::-1])
    assert y.sum() == K.sum()
    mask = np.zeros(shape, np.uint8); mask[4, 5] = 1; mask[0, 0] = 1
    sd = SetDef("BLUR_MASK", "bounds", kernel=K, mask=mask)
    np.testing.assert_array_equal(O.apply_A(shape, sd, x), [0.0, K[1, 2]])


# ------------------------------------------------------------ system matrix
def test_gram_worked_examples():
    g = GOLD["gram_dz_3x1"]
    A = dense_of((3, 1), SetDef("DZ", "bounds"))
    np.testing.assert_array_equal(A.T @ A, np.array(g["matrix"], float))
    g2 = GOLD["system_I_plus_dz"]
    # sets {I-box, D_z-box} with rho = {1 (I set), 1 (D_z set)} and rho_{p+1} -> 0
    C = np.stack([O.apply_C((3, 1), [SetDef("I", "bounds"), SetDef("DZ", "bounds")],
                            [1.0, 1.0, 0.0], np.eye(3)[j]) for j in range(3)], axis=1)
    np.testing.assert_array_equal(C, np.array(g2["matrix"], float))
    np.testing.assert_array_equal(C @ np.eye(3)[0], g2["times_e0"])


@pytest.mark.parametrize("shape", [(5, 4), (3, 4, 3)])
def test_apply_C_matches_dense_assembly(shape):
    """Eq. 23 assembled densely from the operators' matrices"""
    sets = [SetDef("I", "bounds"), SetDef("DZ", "bounds"), SetDef("DX", "card"), SetDef("TV", "l1")]
    if len(shape) == 3:
        sets.append(SetDef("DY", "bounds"))
    else:
        sets.append(_blur_set(shape, sym=True))
    r = np.random.default_rng(3)
    rho = r.uniform(0.1, 3.0, size=len(sets) + 1)
    N = int(np.prod(shape))
    C = rho[-1] * np.eye(N)
    for i, sd in enumerate(sets):
        A = dense_of(shape, sd)
        C += rho[i] * A.T @ A
    for _ in range(3):
        p = r.normal(size=N)
        np.testing.assert_allclose(O.apply_C(shape, sets, rho, p), C @ p, rtol=1e-12, atol=1e-12)
    z = r.normal(size=(20, N))
    assert np.all(np.einsum("ij,jk,ik->i", z, C, z) > 0)   # SPD
    np.testing.assert_allclose(C, C.T, atol=1e-13)


# ------------------------------------------------------------ CG
def _system(shape, seed=5):
    sets = [SetDef("TV", "l1"), SetDef("DZ", "bounds")]
    r = np.random.default_rng(seed)
    rho = r.uniform(0.2, 2.0, size=3)
    N = int(np.prod(shape))
    C = rho[-1] * np.eye(N)
    for i, sd in enumerate(sets):
        A = dense_of(shape, sd)
        C += rho[i] * A.T @ A
    return sets, rho, C


def test_cg_exact_terminates_in_n():
    """exact-arithmetic CG solves an SPD n x n system in <= n steps"""
    shape = (4, 3)
    sets, rho, C = _system(shape)
    b = np.random.default_rng(1).normal(size=12)
    x, it, tol, bd = O.cg(shape, sets, rho, b, np.zeros(12), n_cg=12, eq25=False)
    np.testing.assert_allclose(x, np.linalg.solve(C, b), rtol=1e-9, atol=1e-9)
    assert it <= 12 and bd == 0


def test_cg_eq25_reduces_residual_tenfold():
    """Eq. 25: stop once ||r||/||b|| < 0.1 x the warm-start value"""
    shape = (6, 5)
    sets, rho, C = _system(shape, 9)
    r = np.random.default_rng(2)
    b = r.normal(size=30)
    x0 = r.normal(size=30)
    x, it, tol, bd = O.cg(shape, sets, rho, b, x0, n_cg=100, eq25=True)
    r0 = np.linalg.norm(b - C @ x0) / np.linalg.norm(b)
    r1 = np.linalg.norm(b - C @ x) / np.linalg.norm(b)
    assert tol == pytest.approx(0.1 * r0, rel=1e-12)
    assert r1 < tol and it >= 1
    # one iteration fewer does not reach it (the test is applied before each step)
    x2, it2, _, _ = O.cg(shape, sets, rho, b, x0, n_cg=it - 1, eq25=True)
    assert np.linalg.norm(b - C @ x2) / np.linalg.norm(b) >= tol * (1 - 1e-9)


def test_cg_special_cases():
    """C = rho I converges in one step; warm start at the solution
    takes 0 steps; zero rhs gives x = 0"""
    shape = (3, 3)
    b = np.arange(9.0) + 1
    x, it, _, _ = O.cg(shape, [], [2.0], b, np.zeros(9), n_cg=10, eq25=False)
    np.testing.assert_allclose(x, b / 2.0, rtol=1e-15)
    assert it == 1
    sets, rho, C = _system(shape)
    xs = np.linalg.solve(C, b)
    _, it0, _, _ = O.cg(shape, sets, rho, C @ xs, xs, n_cg=10, eq25=True)
    assert it0 <= 1
    xz, itz, _, _ = O.cg(shape, sets, rho, np.zeros(9), np.ones(9), n_cg=10)
    assert itz == 0 and np.all(xz == 0)


# ------------------------------------------------------------ projectors
def test_projector_worked_examples():
    g = GOLD
    np.testing.assert_array_equal(
        O.project(SetDef("I", "bounds", lo=g["box"]["lo"], hi=g["box"]["hi"]), g["box"]["w"]), g["box"]["y"])
    pd = g["prox_dist"]
    assert O.prox_dist([pd["m"]], pd["rho"], [pd["w"]])[0] == pd["y"]
    for key in ("l1_single", "l1_split"):
        e = g[key]
        np.testing.assert_allclose(O.project(SetDef("I", "l1", sigma=e["sigma"]), e["w"]), e["y"], atol=1e-15)
    e = g["card"]
    np.testing.assert_array_equal(O.project(SetDef("I", "card", k=e["k"]), e["w"]), e["y"])
    e = g["l2_scale"]
    np.testing.assert_allclose(O.project(SetDef("I", "l2", sigma=e["sigma_hi"]), e["w"]), e["y"], rtol=1e-15)
    np.testing.assert_allclose(
        O.project(SetDef("I", "annulus", sigma_lo=0.0, sigma_hi=e["sigma_hi"]), e["w"]), e["y"], rtol=1e-15)
    e = g["annulus_up"]
    np.testing.assert_allclose(
        O.project(SetDef("I", "annulus", sigma_lo=e["sigma_lo"], sigma_hi=e["sigma_hi"]), e["w"]),
        e["y"], rtol=1e-15)
    # reading L7: annulus at 0 -> sigma_l e_1
    np.testing.assert_array_equal(O.project(SetDef("I", "annulus", sigma_lo=2.0, sigma_hi=3.0),
                                            [0.0, 0.0, 0.0]), [2.0, 0.0, 0.0])


def _l1_bruteforce(w, sigma):
    """Euclidean projection onto the l1 ball by KKT support enumeration:
    for each support S, theta = (sum_S |w| - sigma)/|S|; keep supports with
    theta >= 0, |w_j| > theta on S and |w_j| <= theta off S."""
    a = np.abs(w)
    if a.sum() <= sigma:
        return w.copy()
    n = len(w)
    best = None
    for r in range(1, n + 1):
        for S in itertools.combinations(range(n), r):
            S = list(S)
            th = (a[S].sum() - sigma) / len(S)
            off = [j for j in range(n) if j not in S]
            if th >= 0 and np.all(a[S] > th) and np.all(a[off] <= th):
                y = np.sign(w) * np.maximum(a - th, 0.0)
                d = np.linalg.norm(y - w)
                if best is None or d < best[0]:
                    best = (d, y)
    return best[1]


def test_l1_ball_bruteforce():
    r = np.random.default_rng(11)
    for trial in range(150):
        n = int(r.integers(1, 11))
        w = r.normal(size=n) * r.choice([0.1, 1.0, 10.0])
        if trial % 5 == 0:
            w = np.round(w)          # ties
        sigma = float(r.uniform(0, 1.2) * np.abs(w).sum())
        y = O.project(SetDef("I", "l1", sigma=sigma), w)
        np.testing.assert_allclose(y, _l1_bruteforce(w, sigma), rtol=1e-12, atol=1e-12)
        assert np.abs(y).sum() <= sigma * (1 + 1e-12) + 1e-15


def test_cardinality_bruteforce():
    """minimal dropped energy over all C(n,k) supports; ties to lowest index"""
    r = np.random.default_rng(12)
    for trial in range(120):
        n = int(r.integers(1, 11))
        k = int(r.integers(0, n + 1))
        w = r.normal(size=n)
        if trial % 3 == 0:
            w = np.round(w * 2) / 2
        y = O.project(SetDef("I", "card", k=k), w)
        best = min(((w[[j for j in range(n) if j not in S]] ** 2).sum(), S)
                   for S in itertools.combinations(range(n), k))
        assert ((w - y) ** 2).sum() == pytest.approx(best[0], abs=1e-14)
        assert np.count_nonzero(y) <= k
    # tie convention (reading L6)
    np.testing.assert_array_equal(O.project(SetDef("I", "card", k=2), [2.0, -2.0, 1.0, 2.0]),
                                  [2.0, -2.0, 0.0, 0.0])


def test_projector_invariants():
    """idempotence, feasibility, non-expansiveness (convex kinds)"""
    r = np.random.default_rng(13)
    sets = [SetDef("I", "bounds", lo=-0.5, hi=0.7), SetDef("I", "l1", sigma=2.0),
            SetDef("I", "l2", sigma=1.5), SetDef("I", "annulus", sigma_lo=1.0, sigma_hi=2.0),
            SetDef("I", "card", k=3)]
    for sd in sets:
        for _ in range(40):
            a = r.normal(size=9) * 2
            b = r.normal(size=9) * 2
            pa = O.project(sd, a)
            np.testing.assert_allclose(O.project(sd, pa), pa, rtol=1e-12, atol=1e-14)
            if sd.kind == "bounds":
                assert pa.min() >= -0.5 and pa.max() <= 0.7
            if sd.kind == "l1":
                assert np.abs(pa).sum() <= 2.0 * (1 + 1e-12)
            if sd.kind in ("l2", "annulus"):
                radius = sd.sigma if sd.kind == "l2" else sd.sigma_hi
                assert np.linalg.norm(pa) <= radius * (1 + 1e-12)
            if sd.kind == "annulus":
                assert np.linalg.norm(pa) >= 1.0 * (1 - 1e-12)
            if sd.kind == "card":
                assert np.count_nonzero(pa) <= 3
            if sd.kind in ("bounds", "l1", "l2"):
                assert np.linalg.norm(pa - O.project(sd, b)) <= np.linalg.norm(a - b) * (1 + 1e-12)


def test_feasibility_eq26():
    e = GOLD["feas_bounds"]
    assert O.feas(SetDef("I", "bounds", lo=e["lo"], hi=e["hi"]), e["s"]) == pytest.approx(e["r"])
    # reading L19: ||s|| = 0
    assert O.feas(SetDef("I", "bounds", lo=-1, hi=1), [0.0, 0.0]) == 0.0
    assert O.feas(SetDef("I", "bounds", lo=1, hi=2), [0.0, 0.0]) == np.inf
    assert O.feas(SetDef("I", "annulus", sigma_lo=1, sigma_hi=2), [0.0]) == np.inf


# ------------------------------------------------------------ Algorithm 2
def _alg2(dh, dvh, dg, dv, rho=0.7):
    z = np.zeros_like(dh)
    return O.adapt_rho_gamma(dvh, z, dv, z, dh, z, -dg, z, rho)   # y - y0 = -dg


def test_alg2_four_branches():
    """Algorithm 2 case table on constructed vectors whose
    spectral estimates are known in closed form."""
    c = GOLD["alg2_constants"]
    u = np.array([1.0, 2.0, -1.0]); w = np.array([0.5, 0.0, 2.0])
    perp = np.array([2.0, -1.0, 0.0])               # u . perp = 0 -> corr 0
    # alpha: dh = 2u, dvh = 3u  -> corr 1, MG = SD = 1.5 -> ahat = 1.5
    # beta : dg = 4w, dv = 1w   -> corr 1, MG = SD = 0.25 -> bhat = 0.25
    r, g, br = _alg2(2 * u, 3 * u, 4 * w, 1 * w)
    assert br == 0
    assert r == pytest.approx(np.sqrt(1.5 * 0.25), rel=1e-14)
    assert g == pytest.approx(1 + 2 * np.sqrt(1.5 * 0.25) / (1.5 + 0.25), rel=1e-14)
    r, g, br = _alg2(2 * u, 3 * u, 4 * w, perp)       # beta corr = w.perp/...
    assert (br, r, g) == (1, pytest.approx(1.5), c["gamma_alpha_only"])
    r, g, br = _alg2(2 * u, perp, 4 * w, 1 * w)
    assert (br, r, g) == (2, pytest.approx(0.25), c["gamma_beta_only"])
    r, g, br = _alg2(2 * u, perp, 4 * w, np.zeros(3), rho=0.7)   # zero norm -> fails (L17)
    assert (br, r, g) == (3, 0.7, c["gamma_none"])


def test_alg2_sd_branch_and_gamma_two():
    # dh = (1,0), dvh = (1,1): hv = 1, hh = 1, |dvh|^2 = 2 -> corr = 0.707,
    # MG = 1, SD = 2, 2 MG > SD fails -> ahat = SD - MG/2 = 1.5
    z2 = np.zeros(2)
    r, g, br = _alg2(np.array([1.0, 0]), np.array([1.0, 1.0]), z2, z2)
    assert br == 1 and r == pytest.approx(1.5)
    # equal estimates give gamma = 1 + 2a/(2a) = 2 (clamped to 2 - 1e-3 by L15 in PARSDMM)
    u = np.array([1.0, -2.0])
    r, g, br = _alg2(u, 2 * u, u, 2 * u)
    assert br == 0 and g == pytest.approx(2.0, abs=1e-15) and r == pytest.approx(2.0)
    # correlation threshold eps_corr = 0.3: corr 0.25 fails, 0.35 passes
    for corr, ok in ((0.25, False), (0.35, True)):
        dh = np.array([1.0, 0.0]); dvh = np.array([corr, np.sqrt(1 - corr ** 2)])
        _, _, br = _alg2(dh, dvh, z2, z2)
        assert (br == 1) == ok


# ------------------------------------------------------------ PARSDMM end to end
def test_parsdmm_single_box_is_clamp():
    """p = 1, bounds with A = I -> x = clamp(m) (within 1e-4)"""
    m = tiny_model(3, (8, 8))
    sd = SetDef("I", "bounds", lo=2000.0, hi=3500.0)
    r = O.parsdmm((8, 8), [sd], m)
    assert r.converged
    assert O.relres(r.x, np.clip(m, 2000, 3500).ravel()) < 1e-4


def _box_mono_exact(m, lo, hi):
    """projection onto {lo <= x <= hi} with nondecreasing columns in z:
    clip of the per-column isotonic regression (textbook; scipy routine)"""
    out = np.empty_like(m)
    for j in range(m.shape[1]):
        out[:, j] = np.clip(so.isotonic_regression(m[:, j]).x, lo, hi)
    return out


@pytest.mark.parametrize("shape,seed", [((16, 16), 21), ((64, 64), 0)])
def test_parsdmm_box_monotone_vs_isotonic(shape, seed):
    m = tiny_model(seed, shape) if seed else __import__("sip_inputs").c1_model(0, shape)
    sets = [SetDef("I", "bounds", lo=1500.0, hi=4500.0), SetDef("DZ", "bounds", lo=0.0, hi=INF)]
    ref = _box_mono_exact(m, 1500.0, 4500.0)
    r = O.parsdmm(shape, sets, m)
    assert r.converged and r.r_feas.max() < 1e-3
    # production stop (Eq. 28, eps_evol = 1e-2): accurate on the eps_evol scale
    assert O.relres(r.x, ref) < 1e-2
    t = O.parsdmm(shape, sets, m, eps_evol=1e-9, eps_feas=1e-9, n_cg=200, max_iter=20000)
    assert O.relres(t.x, ref) < 1e-6


def _dykstra(m, projs, iters=20000):
    """Algorithm 4: parallel Dykstra with equal weights"""
    p = len(projs)
    x = m.copy()
    v = [m.copy() for _ in range(p)]
    for _ in range(iters):
        y = [P(vi) for P, vi in zip(projs, v)]
        x_new = sum(y) / p
        v = [x_new + vi - yi for vi, yi in zip(v, y)]
        if np.linalg.norm(x_new - x) <= 1e-14 * np.linalg.norm(x):
            x = x_new
            break
        x = x_new
    return x


def test_parsdmm_vs_dykstra_box_mono_l2():
    """box ∩ vertical monotonicity ∩ l2-ball around a center: every set has an
    exact projector, so Algorithm 4 gives the reference projection"""
    shape = (10, 6)
    m = tiny_model(31, shape)
    c0 = np.full(shape, 3000.0)
    rad = 0.6 * np.linalg.norm(m - c0)
    projs = [
        lambda z: np.clip(z, 1500.0, 4500.0),
        lambda z: np.column_stack([so.isotonic_regression(z[:, j]).x for j in range(shape[1])]),
        lambda z: c0 + (z - c0) * min(1.0, rad / np.linalg.norm(z - c0)),
    ]
    ref = _dykstra(m, projs)
    # PARSDMM projects m - c0 (translation invariance of the l2 ball)
    sets = [SetDef("I", "bounds", lo=1500.0 - 3000.0, hi=4500.0 - 3000.0),
            SetDef("DZ", "bounds", lo=0.0, hi=INF), SetDef("I", "l2", sigma=rad)]
    t = O.parsdmm(shape, sets, m - c0, eps_evol=1e-10, eps_feas=1e-10, n_cg=200, max_iter=50000)
    assert O.relres(t.x + c0.ravel(), ref) < 1e-6


def _slsqp_tv(m, shape, sigma, lo, hi, mono=True):
    """exact projection onto bounds ∩ {||TV x||_1 <= sigma} ∩ {D_z x >= 0}
    by scipy SLSQP on the lifted QP (-t <= Dx <= t, sum t <= sigma)"""
    D = dense_of(shape, SetDef("TV", "l1"))
    Dz = dense_of(shape, SetDef("DZ", "bounds"))
    N, M = D.shape[1], D.shape[0]
    m = m.ravel()

    def f(z):
        return 0.5 * np.sum((z[:N] - m) ** 2)

    def fg(z):
        g = np.zeros_like(z); g[:N] = z[:N] - m
        return g

    A_ub = [np.hstack([D, -np.eye(M)]), np.hstack([-D, -np.eye(M)]),
            np.hstack([np.zeros((1, N)), np.ones((1, M))])]
    b_ub = [np.zeros(M), np.zeros(M), [sigma]]
    if mono:
        A_ub.append(np.hstack([-Dz, np.zeros((Dz.shape[0], M))])); b_ub.append(np.zeros(Dz.shape[0]))
    A = np.vstack(A_ub); b = np.concatenate(b_ub)
    cons = [{"type": "ineq", "fun": lambda z: b - A @ z, "jac": lambda z: -A}]
    bounds = [(lo, hi)] * N + [(0, None)] * M
    z0 = np.concatenate([np.clip(m, lo, hi), np.abs(D @ m)])
    res = so.minimize(f, z0, jac=fg, constraints=cons, bounds=bounds, method="SLSQP",
                      options=dict(maxiter=2000, ftol=1e-16))
    return res.x[:N]


@pytest.mark.parametrize("shape,seed", [((4, 4), 41), ((5, 4), 42), ((3, 3, 3), 43)])
def test_parsdmm_tv_convex_vs_qp(shape, seed):
    """bounds ∩ TV-l1 ∩ monotonicity (the C1/C4 set combination) on
    tiny grids: the unique projection from a QP solver"""
    m = tiny_model(seed, shape)
    D = dense_of(shape, SetDef("TV", "l1"))
    sigma = 0.5 * np.abs(D @ m.ravel()).sum()
    ref = _slsqp_tv(m, shape, sigma, 1500.0, 4500.0)
    sets = [SetDef("I", "bounds", lo=1500.0, hi=4500.0), SetDef("TV", "l1", sigma=sigma),
            SetDef("DZ", "bounds", lo=0.0, hi=INF)]
    t = O.parsdmm(shape, sets, m, eps_evol=1e-9, eps_feas=1e-9, n_cg=100, max_iter=100000)
    assert O.relres(t.x, ref) < 1e-5
    r = O.parsdmm(shape, sets, m)
    assert O.relres(r.x, ref) < 2e-2


# ------------------------------------------------------------ multilevel
def test_multilevel_transfers_worked_examples():
    e = GOLD["restrict_2x4"]
    np.testing.assert_array_equal(O.restrict((2, 4), np.array(e["f"], float)), np.array(e["c"], float))
    e = GOLD["interp_2x2_to_3x3"]
    np.testing.assert_allclose(O.interp(np.array(e["c"], float), (3, 3)), np.array(e["f"], float))
    c = np.full((3, 4, 5), 2.5)
    np.testing.assert_allclose(O.interp(c, (5, 7, 9)), 2.5, rtol=1e-15)
    np.testing.assert_allclose(O.restrict((4, 6, 8), np.full((4, 6, 8), 1.25)), 1.25)
    # align-corners: corners map to corners
    r = np.random.default_rng(2).normal(size=(3, 4))
    f = O.interp(r, (5, 7))
    np.testing.assert_allclose(f[::2, ::2], r)


def test_multilevel_one_level_is_single_level():
    p = __import__("sip_inputs").tiny(105, (8, 8), ("bounds", "l1", "slope"))
    x1, st, logs = O.parsdmm_multilevel(p.shape, p.sets, p.m, 1, **p.options)
    r = O.parsdmm(p.shape, p.sets, p.m, **p.options)
    # level-1-only multilevel starts from y = v = 0 -- compare with that init
    r0 = O.parsdmm(p.shape, p.sets, p.m, init=dict(y=[np.zeros(O.op_len(p.shape, s)) for s in p.sets]
                                                    + [np.zeros(p.N)],
                                                    v=None), **p.options)
    np.testing.assert_array_equal(x1, r0.x)
    assert logs[0].iterations == r0.iterations
    assert r.iterations > 0


def test_multilevel_converges_and_is_cheaper():
    """P:533 "the multilevel strategy is much faster": fewer fine-grid CG
    iterations than single level on a 64x64 convex instance"""
    from sip_inputs import c1_model
    m = c1_model(0, (64, 64))
    sets = [SetDef("I", "bounds", lo=1500.0, hi=4500.0), SetDef("DZ", "bounds", lo=0.0, hi=INF)]
    x, st, logs = O.parsdmm_multilevel((64, 64), sets, m, 3)
    single = O.parsdmm((64, 64), sets, m)
    assert logs[0].converged
    assert O.relres(x, _box_mono_exact(m, 1500.0, 4500.0)) < 1e-2
    assert logs[0].cg_total < single.cg_total
    # reading L23: rho and gamma carry over to the next finer level; iteration
    # 1 of a level never adapts (snapshot only), so its logged rho / gamma
    # are the coarser level's final values
    for lf, lc in ((logs[0], logs[1]), (logs[1], logs[2])):
        np.testing.assert_array_equal(lf.rho_trace[0], lc.rho)
        np.testing.assert_array_equal(lf.gamma_trace[0], lc.gamma)
    assert not np.allclose(logs[1].rho, 1e-2)    # the carried values are not the defaults


# ------------------------------------------------------------ per-fiber sets (NEXT-1)
def test_fiber_worked_example():
    """per-row cardinality k = 1 on [[1, 2], [4, 3]] -> [[0, 2], [4, 0]]
    ("applied to each row/column independently"); per column -> [[0, 0], [4, 3]]"""
    np.testing.assert_array_equal(O.project(SetDef("I", "card", k=1, app_mode="x"), [1, 2, 4, 3], shape=(2, 2)),
                                  [0, 2, 4, 0])
    np.testing.assert_array_equal(O.project(SetDef("I", "card", k=1, app_mode="z"), [1, 2, 4, 3], shape=(2, 2)),
                                  [0, 0, 4, 3])


@pytest.mark.parametrize("op,mode,shape", [("I", "x", (5, 4)), ("I", "z", (5, 4)), ("DX", "x", (5, 6)),
                                           ("DX", "z", (5, 6)), ("DZ", "z", (6, 5)), ("DZ", "x", (6, 5)),
                                           ("DY", "x", (3, 4, 5)), ("DX", "z", (4, 3, 5))])
@pytest.mark.parametrize("kind", ["card", "l1", "l2", "annulus"])
def test_fiber_projection_vs_explicit_loop(op, mode, shape, kind):
    """the fiber projector equals an explicit loop over the rows /
    columns of the operator's output field, each projected by the
    whole-vector projector (itself pinned by brute force above)"""
    r = np.random.default_rng(21)
    sd = SetDef(op, kind, k=2, sigma=1.5, sigma_lo=1.0, sigma_hi=1.5, app_mode=mode)
    M = O.op_len(shape, sd)
    L = O.fiber_len(shape, sd)
    nz = shape[0]
    ny = shape[1] if len(shape) == 3 else 1
    nx = shape[-1]
    fz = nz - (op == "DZ")
    fy = ny - (op == "DY")
    fx = nx - (op == "DX")
    assert M == fz * fy * fx and L == (fx if mode == "x" else fz)
    w = r.normal(size=M)
    W = w.reshape(fz, fy, fx)
    ref = np.zeros_like(W)
    whole = SetDef("I", kind, k=2, sigma=1.5, sigma_lo=1.0, sigma_hi=1.5)
    if mode == "x":
        for a in range(fz):
            for b in range(fy):
                ref[a, b, :] = O.project(whole, W[a, b, :])
    else:
        for b in range(fy):
            for c in range(fx):
                ref[:, b, c] = O.project(whole, W[:, b, c])
    np.testing.assert_allclose(O.project(sd, w, shape=shape), ref.ravel(), rtol=0, atol=1e-14)


def test_fiber_bounds_is_separable_and_feasibility():
    """per-row bounds == whole-field bounds (separable set); Eq. 26 of a
    fiber set measures the distance to the per-fiber projection"""
    r = np.random.default_rng(22)
    w = r.normal(size=20)
    a = O.project(SetDef("I", "bounds", lo=-0.3, hi=0.5, app_mode="x"), w, shape=(4, 5))
    b = O.project(SetDef("I", "bounds", lo=-0.3, hi=0.5), w)
    np.testing.assert_array_equal(a, b)
    sd = SetDef("I", "card", k=1, app_mode="x")
    s = np.array([1.0, 2.0, 4.0, 3.0])
    expect = np.linalg.norm([1.0, 0.0, 0.0, 3.0]) / np.linalg.norm(s)
    assert O.feas(sd, s, shape=(2, 2)) == pytest.approx(expect, rel=1e-15)


def test_parsdmm_fiber_l1_vs_dykstra():
    """convex per-row l1 balls (A = I) with bounds: PARSDMM run tightly equals
    Dykstra's algorithm (Algorithm 4) with the exact per-row projector"""
    shape = (6, 8)
    m = tiny_model(33, shape)
    sig = 0.4 * np.abs(m - 3000.0).sum(axis=1).min()
    c0 = np.full(shape, 3000.0)
    row = SetDef("I", "l1", sigma=sig, app_mode="x")
    projs = [lambda z: np.clip(z, 1500.0 - 3000.0, 4500.0 - 3000.0),
             lambda z: O.project(row, z.ravel(), shape=shape).reshape(shape)]
    ref = _dykstra(m - c0, projs)
    sets = [SetDef("I", "bounds", lo=1500.0 - 3000.0, hi=4500.0 - 3000.0), row]
    t = O.parsdmm(shape, sets, m - c0, eps_evol=1e-10, eps_feas=1e-10, n_cg=200, max_iter=50000)
    assert O.relres(t.x, ref.ravel()) < 1e-6
    assert all(np.abs(t.x.reshape(shape)).sum(axis=1) <= sig * (1 + 1e-6))


# ------------------------------------------------------------ hand-derived traces (tests/golden/hand_traces.json)
HT = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "hand_traces.json")))


def _fr(s):
    from fractions import Fraction
    return float(Fraction(s))


def _alg2_trace(max_iter, **opts):
    sets = [SetDef("I", "bounds", lo=0.0, hi=1.0), SetDef("I", "bounds")]
    m = np.full((2, 2), 3.0)
    return O.parsdmm((2, 2), sets, m, want_yv=True, init=dict(rho=[3.0, 0.5, 1.0]),
                     max_iter=max_iter, **opts)


def test_alg2_callsite_hand_trace():
    """Algorithm 2 at its call site: v_hat from the OLD y and v,
    adapt at odd k with a snapshot-only first call, Delta h
    against the k0 snapshot; pinned by a hand-derived 3-iteration trace."""
    e = HT["alg2_callsite_trace"]
    for k in (1, 2, 3):
        r = _alg2_trace(k)
        assert r.iterations == k
        np.testing.assert_allclose(r.x, _fr(e["x"][k - 1]), rtol=0, atol=1e-14)
        np.testing.assert_array_equal(r.cg_per_iter, e["cg"][:k])
    r = _alg2_trace(3)
    np.testing.assert_array_equal(r.branch[0], [-1, -1, -1])   # first call: snapshot only
    np.testing.assert_array_equal(r.branch[1], [-1, -1, -1])   # even k: no adapt
    np.testing.assert_array_equal(r.branch[2], e["branch_k3"])
    np.testing.assert_allclose(r.rho_trace[2], [_fr(s) for s in e["rho_k3"]], rtol=1e-14)
    np.testing.assert_allclose(r.gamma_trace[2], e["gamma_k3"], rtol=1e-14)
    for i in range(3):
        np.testing.assert_allclose(r.y[i], _fr(e["y_k3"][i]), atol=1e-14)
        np.testing.assert_allclose(r.v[i], _fr(e["v_k3"][i]), atol=1e-14)
    # L16: rho_i / rho_{p+1} clamped after the new rho_{p+1}
    r = _alg2_trace(3, rho_ratio_cap=10.0)
    np.testing.assert_allclose(r.rho_trace[2], [_fr(s) for s in e["rho_k3_cap10"]], rtol=1e-14)
    # L15: gamma clamped to gamma_max at the call site
    r = _alg2_trace(3, gamma_max=1.5)
    np.testing.assert_allclose(r.gamma_trace[2], e["gamma_k3_gmax15"], rtol=1e-14)


def test_eq27_history_window_hand_trace():
    """Eq. 27's window of the last s = 5 iterates and the check every 5
    (P:236-246), pinned by a hand-derived trace whose x^k is 5, 3, 1, 1, ..."""
    e = HT["eq27_history_trace"]
    sets = [SetDef("I", "bounds", lo=0.0, hi=1.0)]
    r = O.parsdmm((2, 2), sets, np.full((2, 2), 3.0), max_iter=30, rho0=1.0,
                  init=dict(x=np.full((2, 2), 5.0)))
    assert r.iterations == e["iterations"] and r.converged
    np.testing.assert_array_equal(r.cg_per_iter[:3], e["cg"])
    assert r.r_evol_trace[4] == pytest.approx(e["r_evol_k5"], abs=1e-12)
    assert abs(r.r_evol_trace[9] - e["r_evol_k10"]) < 1e-12
    assert np.isnan(r.r_evol_trace[[0, 1, 2, 3, 5, 6, 7, 8]]).all()   # checked only at k = 5, 10
    np.testing.assert_allclose(r.x, 1.0, atol=1e-12)


def test_prolong_field_shapes():
    """Algorithm 3's transfer of y_i, v_i: each operator field on its own
    shape (reading L23)."""
    e = HT["prolong_fields"]
    cs, fs = tuple(e["coarse"]), tuple(e["fine"])
    for op, key in (("DZ", "dz"), ("DX", "dx"), ("TV", "tv")):
        f = O.prolong_field(cs, fs, op, e[key]["c"])
        np.testing.assert_allclose(f, e[key]["f"], atol=1e-14)
    # I field: constants are preserved on any shape
    np.testing.assert_allclose(O.prolong_field(cs, fs, "I", np.full(4, 7.5)), 7.5, atol=1e-14)


def test_relative_parameter_resolution():
    """relative radii and k resolved from the input m (readings L4, L23)"""
    e = HT["relative_params"]
    shape, m = tuple(e["shape"]), np.array(e["m"], dtype=float)
    s, _, _, _ = O.resolve_set(shape, SetDef("TV", "l1", sigma=0.5, relative=True), m)
    assert s == pytest.approx(e["tv_l1_sigma"], rel=1e-15)
    _, lo, hi, _ = O.resolve_set(shape, SetDef("I", "annulus", sigma_lo=0.9, sigma_hi=1.1, relative=True), m)
    assert lo == pytest.approx(0.9 * np.sqrt(e["annulus_norm_sq"]), rel=1e-15)
    assert hi == pytest.approx(1.1 * np.sqrt(e["annulus_norm_sq"]), rel=1e-15)
    s, _, _, _ = O.resolve_set(shape, SetDef("DZ", "l2", sigma=0.5, relative=True), m)
    assert s * s == pytest.approx(0.25 * e["l2_dz_sigma_sq_over_frac_sq"], rel=1e-14)
    for frac, k in e["card_dx_k"].items():
        _, _, _, kk = O.resolve_set(shape, SetDef("DX", "card", k_frac=float(frac), relative=True), m)
        assert kk == k


# ------------------------------------------------------------ rank / nuclear-norm sets (NEXT-2, Table 1)
def _np_rank(a, r):
    U, s, Vt = np.linalg.svd(a, full_matrices=False)
    return (U[:, :r] * s[:r]) @ Vt[:r]


def _np_nuclear(a, sigma):
    U, s, Vt = np.linalg.svd(a, full_matrices=False)
    if s.sum() <= sigma:
        return a.copy()
    lam = _l1_ball_sorted(s, sigma)
    return (U * lam) @ Vt


def _l1_ball_sorted(s, sigma):
    """projection of a non-negative vector onto {sum <= sigma} by its KKT
    conditions: lam = max(s - theta, 0) with theta the root of sum = sigma
    (bisection, independent of the oracle's sort-based Duchi)"""
    lo, hi = 0.0, float(s.max())
    for _ in range(200):
        th = 0.5 * (lo + hi)
        if np.maximum(s - th, 0).sum() > sigma:
            lo = th
        else:
            hi = th
    return np.maximum(s - 0.5 * (lo + hi), 0)


@pytest.mark.parametrize("shape", [(7, 5), (5, 7), (6, 6), (12, 3)])
def test_svd_values_vs_numpy(shape):
    r = np.random.default_rng(sum(shape))
    a = r.normal(size=shape)
    np.testing.assert_allclose(O.svd_values(a), np.linalg.svd(a, compute_uv=False), rtol=0, atol=1e-13)
    b = np.outer(r.normal(size=shape[0]), r.normal(size=shape[1]))       # rank 1
    sv = O.svd_values(b)
    assert sv[0] == pytest.approx(np.linalg.norm(b), rel=1e-14) and np.all(sv[1:] < 1e-13 * sv[0])


def test_matrix_view_shapes():
    """reading L29: 2D grids one (z, x) matrix, 3D grids one (y, x) matrix per z-plane"""
    assert O.matrix_shape((5, 7), "I") == (5, 7)
    assert O.matrix_shape((5, 7), "DZ") == (4, 7)
    assert O.matrix_shape((5, 7), "DX") == (5, 6)
    assert O.matrix_shape((4, 5, 6), "I") == (5, 6)
    assert O.matrix_shape((4, 5, 6), "DY") == (4, 6)
    assert O.matrix_shape((4, 5, 6), "DZ") == (5, 6)


@pytest.mark.parametrize("shape,op", [((9, 7), "I"), ((7, 9), "DZ"), ((6, 8), "DX"), ((4, 5, 6), "I"),
                                      ((4, 6, 5), "DY")])
def test_rank_projection_is_eckart_young(shape, op):
    """P(A) for {rank <= r} = the truncated SVD (Eckart-Young), per matrix of the view"""
    r = np.random.default_rng(len(shape) + shape[0])
    sd = SetDef(op, "rank", k=2)
    M = O.op_len(shape, sd)
    w = r.normal(size=M)
    y = O.project(sd, w, shape=shape)
    rows, cols = O.matrix_shape(shape, op)
    for o in range(0, M, rows * cols):
        a = w[o:o + rows * cols].reshape(rows, cols)
        np.testing.assert_allclose(y[o:o + rows * cols].reshape(rows, cols), _np_rank(a, 2), atol=1e-12)
        assert np.linalg.matrix_rank(y[o:o + rows * cols].reshape(rows, cols), tol=1e-9) == 2
    np.testing.assert_allclose(O.project(sd, y, shape=shape), y, atol=1e-12)        # idempotent


def test_rank_ties_to_lowest_index():
    """reading L29: equal singular values are ranked by index, so rank 1 of
    diag(2, 2, 1) keeps the first column's direction: diag(2, 0, 0) (a
    diagonal matrix needs no Jacobi rotation, the column order is the
    matrix's own)"""
    a = np.diag([2.0, 2.0, 1.0])
    y = O.project(SetDef("I", "rank", k=1), a.ravel(), shape=(3, 3)).reshape(3, 3)
    np.testing.assert_array_equal(y, np.diag([2.0, 0.0, 0.0]))
    y2 = O.project(SetDef("I", "rank", k=2), a.ravel(), shape=(3, 3)).reshape(3, 3)
    np.testing.assert_array_equal(y2, np.diag([2.0, 2.0, 0.0]))


def test_nuclear_projection_worked_example_and_numpy():
    """diag(3, 2, 1) onto {||A||_* <= 3}: theta = 1, singular values (2, 1, 0)
    (the simplex projection of Table 1's nuclear-norm row); random matrices
    against numpy's SVD with an independent bisection for theta"""
    a = np.diag([3.0, 2.0, 1.0])
    sd = SetDef("I", "nuclear", sigma=3.0)
    y = O.project(sd, a.ravel(), shape=(3, 3)).reshape(3, 3)
    np.testing.assert_allclose(y, np.diag([2.0, 1.0, 0.0]), atol=1e-14)
    r = np.random.default_rng(5)
    for shape in [(8, 5), (5, 8)]:
        b = r.normal(size=shape)
        nuc = np.linalg.svd(b, compute_uv=False).sum()
        sd = SetDef("I", "nuclear", sigma=0.4 * nuc)
        y = O.project(sd, b.ravel(), shape=shape).reshape(shape)
        np.testing.assert_allclose(y, _np_nuclear(b, 0.4 * nuc), atol=1e-10)
        assert np.linalg.svd(y, compute_uv=False).sum() <= 0.4 * nuc * (1 + 1e-12)
        inside = SetDef("I", "nuclear", sigma=2 * nuc)
        np.testing.assert_allclose(O.project(inside, b.ravel(), shape=shape), b.ravel(), atol=1e-15)


def test_nuclear_relative_radius():
    """relative sigma of a nuclear-norm set = frac x the nuclear norm of A m
    (summed over the matrices of the view), reading L23/L29"""
    r = np.random.default_rng(9)
    m = r.normal(size=(6, 5))
    sig, _, _, _ = O.resolve_set((6, 5), SetDef("I", "nuclear", sigma=0.5, relative=True), m)
    assert sig == pytest.approx(0.5 * np.linalg.svd(m, compute_uv=False).sum(), rel=1e-13)


def test_parsdmm_nuclear_box_vs_dykstra():
    """box ∩ nuclear-norm ball (both convex, exact projectors): PARSDMM's
    tightly converged point equals parallel Dykstra's (Algorithm 4)"""
    shape = (8, 6)
    r = np.random.default_rng(13)
    m = r.normal(size=shape) * 2.0
    nuc = np.linalg.svd(m, compute_uv=False).sum()
    sig = 0.5 * nuc
    projs = [lambda z: np.clip(z, -1.5, 1.5), lambda z: _np_nuclear(z, sig)]
    ref = _dykstra(m, projs)
    sets = [SetDef("I", "bounds", lo=-1.5, hi=1.5), SetDef("I", "nuclear", sigma=sig)]
    t = O.parsdmm(shape, sets, m, eps_evol=1e-10, eps_feas=1e-10, n_cg=50, max_iter=50000)
    assert O.relres(t.x, ref) < 1e-6


# ------------------------------------------------------------ orthogonal-transform sets (NEXT-3)
@pytest.mark.parametrize("shape", [(5, 7), (8, 8), (3, 4, 5)])
def test_dct_is_scipy_orthonormal_dct2(shape):
    """the oracle's DCT (its own O(n^2) loops) against scipy's dctn(norm='ortho')
    (a library routine), its inverse, and Parseval (orthogonality)"""
    import scipy.fft as F
    r = np.random.default_rng(len(shape))
    x = r.normal(size=shape)
    c = O.dct(shape, x)
    np.testing.assert_allclose(c.reshape(shape), F.dctn(x, norm="ortho"), atol=1e-13)
    np.testing.assert_allclose(O.dct(shape, c, inverse=True).reshape(shape), x, atol=1e-13)
    assert np.linalg.norm(c) == pytest.approx(np.linalg.norm(x), rel=1e-14)
    const = np.full(shape, 2.0)
    cc = O.dct(shape, const)
    assert cc[0] == pytest.approx(2.0 * np.sqrt(np.prod(shape)), rel=1e-14) and np.abs(cc[1:]).max() < 1e-12


def test_dct_l1_projection_closed_form():
    """P_V(x) = D^T P_l1(D x): feasible, idempotent, and equal to the
    projection computed with scipy's DCT and an independent l1-ball bisection"""
    import scipy.fft as F
    shape = (6, 10)
    r = np.random.default_rng(3)
    x = r.normal(size=shape)
    n1 = np.abs(F.dctn(x, norm="ortho")).sum()
    sd = SetDef("I", "dct_l1", sigma=0.3 * n1)
    y = O.project(sd, x.ravel(), shape=shape)
    c = F.dctn(x, norm="ortho").ravel()
    lam = _l1_ball_sorted(np.abs(c), 0.3 * n1)
    ref = F.idctn((np.sign(c) * lam).reshape(shape), norm="ortho").ravel()
    np.testing.assert_allclose(y, ref, atol=1e-9)
    assert np.abs(F.dctn(y.reshape(shape), norm="ortho")).sum() <= 0.3 * n1 * (1 + 1e-12)
    np.testing.assert_allclose(O.project(sd, y, shape=shape), y, atol=1e-12)
    s, _, _, _ = O.resolve_set(shape, SetDef("I", "dct_l1", sigma=0.3, relative=True), x)
    assert s == pytest.approx(0.3 * n1, rel=1e-13)


def test_parsdmm_box_dct_l1_vs_dykstra():
    """box ∩ {||D x||_1 <= sigma}: PARSDMM (the transform kept inside the set,
    A = I) reaches parallel Dykstra's point (Algorithm 4)"""
    import scipy.fft as F
    shape = (8, 6)
    r = np.random.default_rng(17)
    m = r.normal(size=shape) * 3.0
    sig = 0.4 * np.abs(F.dctn(m, norm="ortho")).sum()

    def p_dct(z):
        c = F.dctn(z, norm="ortho")
        lam = _l1_ball_sorted(np.abs(c).ravel(), sig).reshape(shape)
        return F.idctn(np.sign(c) * lam, norm="ortho")
    ref = _dykstra(m, [lambda z: np.clip(z, -2.0, 2.0), p_dct])
    sets = [SetDef("I", "bounds", lo=-2.0, hi=2.0), SetDef("I", "dct_l1", sigma=sig)]
    t = O.parsdmm(shape, sets, m, eps_evol=1e-10, eps_feas=1e-10, n_cg=50, max_iter=50000)
    assert O.relres(t.x, ref) < 1e-6


# ------------------------------------------------------------ Algorithm 4 comparator (NEXT-4, Fig. 1)
def test_oracle_dykstra_matches_algorithm4_with_exact_projectors():
    """the oracle's parallel Dykstra (PARSDMM sub-problems for A != I) against
    Algorithm 4 with exact projectors (box, clip(PAVA) for D_z x >= 0):
    same point; the counters are the paper's"""
    shape = (8, 6)
    m = tiny_model(33, shape)
    lo, hi = float(np.percentile(m, 10)), float(np.percentile(m, 90))
    sets = [SetDef("I", "bounds", lo=lo, hi=hi), SetDef("DZ", "bounds", lo=0.0, hi=INF)]
    ref = _dykstra(m, [lambda z: np.clip(z, lo, hi),
                       lambda z: np.column_stack([so.isotonic_regression(z[:, j]).x for j in range(shape[1])])])
    d = O.dykstra(shape, sets, m, max_outer=3000, tol=1e-13, eps_evol=1e-12, eps_feas=1e-12, n_cg=100,
                  max_iter=20000)
    assert O.relres(d["x"], ref) < 1e-6
    assert (d["cg_max"] > 0).all() and (d["l1_proj"] == 0).all()
    assert (d["inner_iters"][:, 0] == 1).all()          # A = I: one projection, no CG


def test_oracle_dykstra_counts_l1_projections():
    """with a TV l1 set, every outer iteration projects onto the l1 ball as
    often as the TV sub-problem iterates"""
    shape = (8, 8)
    m = tiny_model(34, shape)
    sets = [SetDef("I", "bounds", lo=float(m.min()) + 50, hi=float(m.max()) - 50),
            SetDef("TV", "l1", sigma=0.5, relative=True)]
    d = O.dykstra(shape, sets, m, max_outer=5, tol=0.0)
    assert d["iterations"] == 5
    np.testing.assert_array_equal(d["l1_proj"], d["inner_iters"][:, 1])
    assert (d["l1_proj"] >= 1).all()


def _haar_matrix(L):
    """the orthonormal Haar matrix by its Kronecker recursion (a closed form,
    not the oracle's pyramid): H_1 = [1], H_2n = [H_n (x) [1, 1]; I_n (x) [1, -1]] / sqrt(2)"""
    H = np.ones((1, 1))
    while H.shape[0] < L:
        n = H.shape[0]
        H = np.vstack([np.kron(H, [1.0, 1.0]), np.kron(np.eye(n), [1.0, -1.0])]) / np.sqrt(2.0)
    return H


def _haar_sep(x):
    """the separable transform: the Haar matrix applied along every axis"""
    y = np.asarray(x, dtype=np.float64)
    for ax in range(y.ndim):
        y = np.moveaxis(np.tensordot(_haar_matrix(y.shape[ax]), np.moveaxis(y, ax, 0), axes=1), 0, ax)
    return y


@pytest.mark.parametrize("shape", [(4, 4), (8, 16), (2, 4, 8)])
def test_haar_against_kronecker_matrix(shape):
    """the oracle's Haar pyramid ("wavelet", reading L30) against the
    Kronecker-recursion Haar matrix along every axis, the inverse, Parseval"""
    r = np.random.default_rng(sum(shape))
    x = r.normal(size=shape)
    c = O.haar(shape, x)
    np.testing.assert_allclose(c.reshape(shape), _haar_sep(x), atol=1e-13)
    np.testing.assert_allclose(O.haar(shape, c, inverse=True).reshape(shape), x, atol=1e-13)
    assert np.linalg.norm(c) == pytest.approx(np.linalg.norm(x), rel=1e-14)


def test_haar_worked_examples():
    """4 x 4 by hand: a constant 1 gives the single coefficient sqrt(16) = 4;
    x = e_(0,0) - e_(0,1): the row step gives d_1[0] = (1 - (-1)) / sqrt(2) =
    sqrt(2) at x-position 2, then column 2 = (sqrt(2), 0, 0, 0) -> a = (1, 0),
    d = (1, 0) -> [1/sqrt(2), 1/sqrt(2), 1, 0]"""
    c = O.haar((4, 4), np.ones(16)).reshape(4, 4)
    ref = np.zeros((4, 4))
    ref[0, 0] = 4.0
    np.testing.assert_allclose(c, ref, atol=1e-15)
    x = np.zeros((4, 4))
    x[0, 0], x[0, 1] = 1.0, -1.0
    c = O.haar((4, 4), x).reshape(4, 4)
    ref = np.zeros((4, 4))
    ref[:, 2] = [np.sqrt(0.5), np.sqrt(0.5), 1.0, 0.0]
    np.testing.assert_allclose(c, ref, atol=1e-15)


def test_haar_l1_projection_closed_form_and_dykstra():
    """P_V(x) = H^T P_l1(H x) with the Kronecker Haar matrix and an
    independent l1-ball projection; relative sigma from ||H m||_1; PARSDMM
    box + Haar-l1 reaches parallel Dykstra's point (Algorithm 4)"""
    shape = (8, 16)
    r = np.random.default_rng(23)
    x = r.normal(size=shape)
    n1 = np.abs(_haar_sep(x)).sum()
    sd = SetDef("I", "haar_l1", sigma=0.3 * n1)
    y = O.project(sd, x.ravel(), shape=shape)
    c = _haar_sep(x).ravel()
    lam = _l1_ball_sorted(np.abs(c), 0.3 * n1)
    Hz, Hx = _haar_matrix(shape[0]), _haar_matrix(shape[1])
    ref = (Hz.T @ (np.sign(c) * lam).reshape(shape) @ Hx).ravel()
    np.testing.assert_allclose(y, ref, atol=1e-9)
    np.testing.assert_allclose(O.project(sd, y, shape=shape), y, atol=1e-12)
    s, _, _, _ = O.resolve_set(shape, SetDef("I", "haar_l1", sigma=0.3, relative=True), x)
    assert s == pytest.approx(0.3 * n1, rel=1e-13)
    m = r.normal(size=shape) * 3.0
    sig = 0.4 * np.abs(_haar_sep(m)).sum()

    def p_haar(z):
        cz = _haar_sep(z)
        lz = _l1_ball_sorted(np.abs(cz).ravel(), sig).reshape(shape)
        return Hz.T @ (np.sign(cz) * lz) @ Hx
    dref = _dykstra(m, [lambda z: np.clip(z, -2.0, 2.0), p_haar])
    sets = [SetDef("I", "bounds", lo=-2.0, hi=2.0), SetDef("I", "haar_l1", sigma=sig)]
    t = O.parsdmm(shape, sets, m, eps_evol=1e-10, eps_feas=1e-10, n_cg=50, max_iter=50000)
    assert O.relres(t.x, dref) < 1e-6
