"""Orthogonal-transform l1 sets: {x :
||D x||_1 <= sigma} with D the grid's orthonormal DCT-II or full-depth Haar
wavelet transform (reading L30), projected as
D^T P_l1(D x) (the transform kept inside the set, A = I).  GPU against the
oracle: sip_project_set (1e-5 fp32, 1e-10 fp64) and PARSDMM end to end
(tiny fp64: exact iteration / CG counts; fp32 within 1e-3).  Marked gpu."""
import numpy as np
import pytest

import oracle as O
import sip_inputs as G
from sip_inputs import SetDef

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1902_09699_b200 import Grid  # noqa: E402

TD = {"f32": torch.float32, "f64": torch.float64}
TOL = {"f32": 1e-5, "f64": 1e-10}


def mk(shape, sets, dtype):
    g = Grid(shape, None, dtype)
    for sd in sets:
        g.add_set(sd)
    return g


TRANSFORM = {"dct_l1": O.dct, "haar_l1": O.haar}


@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("kind,shape", [("dct_l1", (48, 64)), ("dct_l1", (96, 32)), ("dct_l1", (6, 20, 16)),
                                        ("haar_l1", (32, 64)), ("haar_l1", (128, 16)), ("haar_l1", (8, 16, 32))])
def test_project_set_dct(dtype, kind, shape):
    r = np.random.default_rng(shape[0])
    w = r.normal(size=int(np.prod(shape))) * 5.0
    n1 = np.abs(TRANSFORM[kind](shape, w)).sum()
    sd = SetDef("I", kind, sigma=0.25 * n1)
    g = mk(shape, [sd], dtype)
    m = torch.zeros(shape, dtype=TD[dtype], device="cuda")
    x = torch.empty_like(m)
    g.project(m, x, max_iter=2)
    wd = torch.tensor(w, dtype=TD[dtype], device="cuda")
    y = torch.empty_like(wd)
    g.project_set(0, wd, y)
    ref = O.project(sd, wd.double().cpu().numpy(), shape=shape)
    assert O.relres(y.double().cpu().numpy(), ref) <= TOL[dtype]
    g.close()


def _prob(shape, dtype, kind="dct_l1"):
    m = G.tiny_model(160 + len(shape), shape)
    sets = [SetDef("I", "bounds", lo=float(m.min()) + 100.0, hi=float(m.max()) - 100.0),
            SetDef("I", kind, sigma=0.6, relative=True)]
    return G.Problem("dct", shape, dtype, m, sets, options=dict(G.DEFAULT_OPTIONS))


@pytest.mark.parametrize("kind,shape", [("dct_l1", (16, 12)), ("dct_l1", (4, 8, 6)), ("haar_l1", (16, 8)),
                                        ("haar_l1", (4, 8, 8))])
def test_parsdmm_dct_fp64_exact(kind, shape):
    prob = _prob(shape, "f64", kind)
    g = mk(shape, prob.sets, "f64")
    m = torch.tensor(prob.m, dtype=torch.float64, device="cuda")
    x = torch.empty_like(m)
    res, st = g.project(m, x, max_iter=200, tol=1e-3)
    lg = g.get_log(200)
    ref = O.parsdmm(shape, prob.sets, prob.m, **prob.options)
    assert res["iterations"] == ref.iterations
    np.testing.assert_array_equal(lg["cg"][: ref.iterations], ref.cg_per_iter)
    np.testing.assert_array_equal(lg["branch"][: ref.iterations], ref.branch)
    assert O.relres(x.cpu().numpy(), ref.x) < 1e-8
    g.close()


@pytest.mark.parametrize("kind,shape", [("dct_l1", (64, 96)), ("haar_l1", (64, 128))])
def test_parsdmm_dct_fp32(kind, shape):
    prob = _prob(shape, "f32", kind)
    g = mk(shape, prob.sets, "f32")
    m = torch.tensor(prob.m, dtype=torch.float32, device="cuda")
    x = torch.empty_like(m)
    g.project(m, x, max_iter=200, tol=1e-3)
    o = dict(prob.options, cg_tol_floor=10 * float(np.finfo(np.float32).eps))
    ref = O.parsdmm(shape, prob.sets, prob.m, **o)
    assert O.relres(x.double().cpu().numpy(), ref.x) < 1e-3
    g.close()


def test_dct_refusals():
    g = Grid((16, 16), None, "f32")
    with pytest.raises(Exception):
        g.add_set(SetDef("DZ", "dct_l1", sigma=1.0))
    g.close()
    g = Grid((16, 12), None, "f32")
    with pytest.raises(Exception):
        g.add_set(SetDef("I", "haar_l1", sigma=1.0))   # 12 is not a power of two
    g.close()
