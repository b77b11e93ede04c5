"""Per-fiber application modes (NEXT-1; a simple set's
projection applied to each row / column of the operator output on its own)
on the GPU (k_fiber, sip_fiber.cuh) against the oracle's per-fiber
projectors (oracle/sipref.c sipref_project, app_mode 1 / 2).

Bars: cardinality supports and kept values exact;
l1 relative L2 <= 10 x the per-kernel tolerance; tiny fp64 end-to-end runs
with identical iteration counts, CG counts and Algorithm-2 branches.
"""
import numpy as np
import pytest

import oracle as O
import sip_inputs as G
from sip_inputs import SetDef

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1902_09699_b200 import Grid, SipError, grid_for  # noqa: E402

TD = {"f32": torch.float32, "f64": torch.float64}
TOL = {"f32": 1e-5, "f64": 1e-12}


def dev(a, dtype):
    return torch.tensor(np.ascontiguousarray(a), dtype=TD[dtype], device="cuda")


def host(t):
    return t.detach().double().cpu().numpy()


# (shape, op, mode): nx a multiple of 4 (16-byte lanes, the vectorised path);
# ragged fiber counts, fibers longer than the CTA, pad fibers (DZ x-fibers,
# DY rows, DX columns) and 2D / 3D
CASES = [
    ((24, 64), "DX", "x"),
    ((5, 4, 32), "DX", "x"),       # 31-entry fibers: one entry per lane
    ((4, 8, 200), "DZ", "x"),      # E = 8 lanes' entries
    ((300, 40), "DZ", "z"),        # 299-entry columns (E = 16), ragged column tile
    ((64, 3, 36), "I", "z"),
    ((24, 64), "DZ", "x"),
    ((24, 64), "I", "z"),
    ((37, 100), "DZ", "z"),
    ((37, 100), "DX", "z"),
    ((6, 10, 12), "DY", "x"),
    ((6, 10, 12), "DY", "z"),
    ((9, 5, 1300), "DX", "x"),     # 1299-entry fibers: 5+ entries per thread
    ((700, 8), "I", "z"),          # 700-entry columns
]


def _case(shape, op, mode, kind, dtype, seed, ties=False):
    sd = SetDef(op, kind, app_mode=mode)
    L = O.fiber_len(shape, sd)
    M = O.op_len(shape, sd)
    r = np.random.default_rng(seed)
    w = r.normal(size=M) * r.choice([0.01, 1.0, 100.0])
    if ties:
        w = np.round(w * 2) / 2
    nf = M // L
    fib = (w.reshape(nf, L) if mode == "x" else w.reshape(L, nf).T)
    if kind == "card":
        sd.k = max(1, int(0.3 * L))
    elif kind in ("l2", "annulus"):
        if kind == "annulus":   # a zero fiber: the annulus maps it to sigma_lo e_1 (L7)
            if mode == "x":
                w[:L] = 0.0
            else:
                w[0::nf] = 0.0
            fib = (w.reshape(nf, L) if mode == "x" else w.reshape(L, nf).T)
        n2 = np.sort(np.linalg.norm(fib, axis=1))
        sd.sigma = float(n2[len(n2) // 2])
        sd.sigma_lo, sd.sigma_hi = float(n2[len(n2) // 3]), float(n2[2 * len(n2) // 3])
    else:
        nf = M // L
        # sigma between the smallest and largest fiber l1 norm: both the
        # inside and the soft-threshold branches are taken
        fib = w.reshape(nf, L) if mode == "x" else w.reshape(L, nf).T
        n1 = np.sort(np.abs(fib).sum(axis=1))
        sd.sigma = float(n1[len(n1) // 3])
    return sd, w


@pytest.mark.parametrize("path", ["warp", "sort"])
@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("kind", ["card", "card_ties", "l1", "l2", "annulus"])
@pytest.mark.parametrize("shape,op,mode", CASES)
def test_project_set_per_fiber(shape, op, mode, kind, dtype, path, monkeypatch):
    """path "warp": k_fiberw (bitwise threshold search, fibers <= 512);
    "sort": k_fiber (bitonic sort, SIP_FIBER_SORT=1); fibers longer than
    512 take the sort kernel on both"""
    if path == "sort":
        monkeypatch.setenv("SIP_FIBER_SORT", "1")
    base = "card" if kind.startswith("card") else kind
    sd, w = _case(shape, op, mode, base, dtype, 7 + len(shape) + len(op), ties=kind == "card_ties")
    g = Grid(shape, None, dtype)
    g.add_set(sd)
    m = dev(np.zeros(shape), dtype)
    x = torch.empty_like(m)
    g.project(m, x, max_iter=1)
    wd = dev(w, dtype)
    wr = host(wd)
    y = torch.empty_like(wd)
    g.project_set(0, wd, y)
    ref = O.project(sd, wr, shape=shape)
    yh = host(y)
    g.close()
    if base == "card":
        np.testing.assert_array_equal(yh != 0, ref != 0)
        np.testing.assert_array_equal(yh, ref)
    else:
        assert O.relres(yh, ref) <= TOL[dtype], O.relres(yh, ref)


def test_card_k_at_least_fiber_length_keeps_all():
    shape = (8, 16)
    sd = SetDef("DX", "card", k=15, app_mode="x")
    w = np.random.default_rng(3).normal(size=O.op_len(shape, sd))
    g = Grid(shape, None, "f64")
    g.add_set(sd)
    m = dev(np.zeros(shape), "f64")
    g.project(m, torch.empty_like(m), max_iter=1)
    y = torch.empty(w.size, dtype=torch.float64, device="cuda")
    g.project_set(0, dev(w, "f64"), y)
    np.testing.assert_array_equal(host(y), w)
    g.close()


FIBER_TINY = [
    (100, (8, 12), ("bounds", "l1_rows", "slope")),
    (100, (12, 8), ("bounds", "l1_rows", "slope")),
    (100, (8, 8), ("bounds", "card_rows")),
    (100, (4, 4, 8), ("bounds", "card_cols", "l1_rows")),
    (100, (8, 8), ("bounds", "l1_cols", "slope")),
    (100, (6, 8), ("bounds", "l1", "card_cols")),
    (100, (4, 4, 8), ("bounds", "l1_cols", "card_rows")),
    (100, (8, 12), ("bounds", "card_rows", "l1_rows")),
    (100, (8, 12), ("bounds", "l2_rows", "slope")),
    (100, (8, 8), ("bounds", "ann_cols", "l1_rows")),
    (100, (4, 4, 8), ("bounds", "l2_rows", "card_cols")),
]


@pytest.mark.parametrize("path", ["warp", "sort"])
@pytest.mark.parametrize("seed,shape,kinds", FIBER_TINY)
def test_tiny_fiber_control_flow(seed, shape, kinds, path, monkeypatch):
    if path == "sort":
        monkeypatch.setenv("SIP_FIBER_SORT", "1")
    prob = G.tiny(seed, shape, kinds)
    g = grid_for(prob)
    m = dev(prob.m, "f64")
    x = torch.empty_like(m)
    res, st = g.project(m, x, max_iter=200, tol=1e-3)
    log = g.get_log(200)
    ref = O.parsdmm(prob.shape, prob.sets, prob.m, **prob.options)
    it = ref.iterations
    if not ref.converged:
        # 200 iterations of a non-converging run amplify rounding-order
        # differences (measured: first CG-count difference after iteration
        # 100 with cardinality / l1 fibers, after 50 with per-fiber l2 norms
        # summed in another order): the control flow is compared on the
        # first 50 iterations, the run length exactly
        assert res["iterations"] == it and not res["converged"]
        it = 50
    else:
        assert res["iterations"] == it
        assert res["converged"]
        assert O.relres(host(x), ref.x) < 1e-6
    np.testing.assert_array_equal(log["cg"][:it], ref.cg_per_iter[:it])
    np.testing.assert_array_equal(log["branch"][:it], ref.branch[:it])
    g.close()


def test_fiber_fp32_medium_run():
    """fp32 on a 96 x 256 layered model: per-row cardinality of the lateral
    derivative and per-column l1 of the model with bounds and a slope set;
    final x within 1e-3 of the fp64 oracle (decisions in fp32, reading L27)"""
    shape = (96, 256)
    m = G.tiny_model(11, shape)
    sets = [SetDef("I", "bounds", lo=1500.0, hi=4500.0),
            SetDef("DZ", "bounds", lo=0.0, hi=G.INF),
            SetDef("DX", "card", k_frac=0.5, relative=True, app_mode="x"),
            SetDef("I", "l1", sigma=2600.0 * shape[0], app_mode="z")]
    opts = dict(G.DEFAULT_OPTIONS)
    prob = G.Problem("fib32", shape, "f32", m, sets, options=opts)
    g = grid_for(prob)
    md = dev(m, "f32")
    x = torch.empty_like(md)
    res, st = g.project(md, x, max_iter=150, tol=1e-3)
    o = dict(opts)
    o["cg_tol_floor"] = 10 * float(np.finfo(np.float32).eps)
    ref = O.parsdmm(shape, sets, host(md), max_iter=150, **{k: v for k, v in o.items() if k != "max_iter"})
    assert O.relres(host(x), ref.x) < 1e-3
    g.close()


def test_fiber_refused_configurations():
    with pytest.raises(SipError):
        g = Grid((8, 8), None, "f64")
        g.add_set(SetDef("TV", "card", k=2, app_mode="x"))          # two-block operator
    with pytest.raises(SipError):
        g = Grid((8, 8), None, "f64")
        g.add_set(SetDef("DX", "l2", sigma=0.5, relative=True, app_mode="x"))   # radii per fiber: absolute
    with pytest.raises(SipError):
        g = Grid((8, 8), None, "f64")
        g.add_set(SetDef("DX", "l1", sigma=0.5, relative=True, app_mode="x"))


# ---------------------------------------------------------------- z slabs
# x-fibers lie in one plane, so they shard with the z slabs (option
# "virtual_ranks": G slabs on one device through the multi-GPU code path);
# each rank's fiber sums join pass 2's gathered reduction.
SLAB_FIBER = [
    (100, (8, 12), ("bounds", "card_rows", "l1_rows"), 3),
    (100, (12, 8), ("bounds", "l1_rows", "slope"), 2),
    (100, (4, 4, 8), ("bounds", "card_rows"), 2),
    (100, (8, 8), ("bounds", "card_rows"), 4),
]


@pytest.mark.parametrize("seed,shape,kinds,ranks", SLAB_FIBER)
def test_slab_x_fibers_control_flow(seed, shape, kinds, ranks):
    prob = G.tiny(seed, shape, kinds)
    ref = O.parsdmm(prob.shape, prob.sets, prob.m, **prob.options)
    g = grid_for(prob)
    g.set_option("virtual_ranks", ranks)
    m = dev(prob.m, "f64")
    x = torch.empty_like(m)
    res, st = g.project(m, x, max_iter=200, tol=1e-3)
    log = g.get_log(200)
    it = ref.iterations
    assert res["iterations"] == it
    lim = it if ref.converged else 50   # see test_tiny_fiber_control_flow
    np.testing.assert_array_equal(log["cg"][:lim], ref.cg_per_iter[:lim])
    np.testing.assert_array_equal(log["branch"][:lim], ref.branch[:lim])
    if ref.converged:
        assert O.relres(host(x), ref.x) < 1e-6
    g.close()


def test_slab_x_fibers_fp32_matches_single_rank():
    shape = (40, 24, 64)
    m = G.tiny_model(21, shape)
    sets = [SetDef("I", "bounds", lo=1500.0, hi=4500.0),
            SetDef("DZ", "bounds", lo=0.0, hi=G.INF),
            SetDef("DX", "card", k_frac=0.5, relative=True, app_mode="x"),
            SetDef("DY", "l1", sigma=150.0 * shape[2], app_mode="x")]
    prob = G.Problem("fibslab", shape, "f32", m, sets, options=dict(G.DEFAULT_OPTIONS))
    xs = []
    for ranks in (1, 4):
        g = grid_for(prob)
        if ranks > 1:
            g.set_option("virtual_ranks", ranks)
        g.set_option("fixed_work", 1)
        md = dev(m, "f32")
        x = torch.empty_like(md)
        g.project(md, x, max_iter=20, tol=1e-3)
        xs.append(host(x))
        g.close()
    assert O.relres(xs[1], xs[0]) < 1e-5


def test_slab_z_fibers_refused():
    prob = G.tiny(100, (8, 8), ("bounds", "card_cols"))
    g = grid_for(prob)
    g.set_option("virtual_ranks", 2)
    m = dev(prob.m, "f64")
    with pytest.raises(SipError):
        g.project(m, torch.empty_like(m), max_iter=5, tol=1e-3)
    g.close()


# ---------------------------------------------------------------- multilevel
@pytest.mark.parametrize("shape,kinds", [
    ((16, 16), ("bounds", "card_rows", "l1_rows")),
    ((16, 16), ("bounds", "l1_cols", "slope")),
    ((8, 8, 16), ("bounds", "card_rows", "slope")),
])
def test_multilevel_with_fibers(shape, kinds):
    """Algorithm 3 with per-fiber sets: each level's fibers have that
    level's length (relative k from it, reading L28); per-level iteration
    and CG counts equal the oracle's while the levels converge"""
    prob = G.tiny(120, shape, kinds)
    g = grid_for(prob)
    m = dev(prob.m, "f64")
    x = torch.empty_like(m)
    per, st = g.project_multilevel(m, x, 2, max_iter=200, tol=1e-3)
    xo, sto, logs = O.parsdmm_multilevel(prob.shape, prob.sets, prob.m, 2, **prob.options)
    all_conv = True
    for l in (1, 0):
        assert per[l]["iterations"] == logs[l].iterations, (l, per[l]["iterations"], logs[l].iterations)
        if not logs[l].converged:
            all_conv = False
            break
        assert per[l]["cg_iterations"] == logs[l].cg_total
    assert O.relres(host(x), xo) < (1e-6 if all_conv else 1e-3)
    g.close()
