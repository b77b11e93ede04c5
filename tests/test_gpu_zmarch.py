"""Parity of the z-marching CG kernels (sip_zmarch.cuh) -- used for 3D grids
whose x rows split into whole warps of 16-byte chunks (nx % 128 == 0 for
fp32, nx % 64 == 0 for fp64).  Same arithmetic as the other CG kernels, so
the same bars: CG iterations equal and x within 1e-4 (fp32) / 1e-10 (fp64)
of the oracle's CG; end to end identical control flow in fp64."""
import numpy as np
import pytest

import oracle as O
import sip_inputs as G
from sip_inputs import SetDef

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1902_09699_b200 import Grid, grid_for  # noqa: E402

TD = {"f32": torch.float32, "f64": torch.float64}


@pytest.mark.parametrize("dtype,shape", [("f32", (10, 16, 128)), ("f32", (7, 8, 256)), ("f32", (5, 24, 1024)),
                                         ("f64", (9, 8, 64)), ("f64", (6, 16, 128))])
@pytest.mark.parametrize("eq25", [True, False])
def test_cg_zmarch(dtype, shape, eq25):
    sets = [SetDef("TV", "l1"), SetDef("DZ", "bounds"), SetDef("DY", "bounds")]
    g = Grid(shape, None, dtype)
    for sd in sets:
        g.add_set(sd)
    r = np.random.default_rng(5)
    rho = r.uniform(0.1, 3.0, size=len(sets) + 1)
    b = torch.tensor(r.normal(size=shape), dtype=TD[dtype], device="cuda")
    x0 = torch.tensor(r.normal(size=shape), dtype=TD[dtype], device="cuda")
    x = x0.clone()
    it = g.cg(rho, b, x, n_cg=20, eq25=eq25)
    xr, itr, tol, bd = O.cg(shape, sets, rho, b.double().cpu().numpy(), x0.double().cpu().numpy(),
                            n_cg=20, eq25=eq25)
    assert it == itr
    assert O.relres(x.double().cpu().numpy(), xr) <= (1e-4 if dtype == "f32" else 1e-10)


@pytest.mark.parametrize("seed,shape,kinds", [
    (160, (6, 8, 64), ("bounds", "l1", "slope")),
    (161, (5, 16, 64), ("bounds", "l1", "slope", "cardz", "annulus")),
])
def test_tiny_zmarch_bitexact(seed, shape, kinds):
    prob = G.tiny(seed, shape, kinds)
    g = grid_for(prob)
    m = torch.tensor(prob.m, dtype=torch.float64, device="cuda")
    x = torch.empty_like(m)
    res, st = g.project(m, x, max_iter=200, tol=1e-3)
    log = g.get_log(200)
    ref = O.parsdmm(prob.shape, prob.sets, prob.m, **prob.options)
    it = ref.iterations
    assert res["iterations"] == it
    np.testing.assert_array_equal(log["cg"][:it], ref.cg_per_iter)
    np.testing.assert_array_equal(log["branch"][:it], ref.branch)
    assert O.relres(x.cpu().numpy(), ref.x) < 1e-6
