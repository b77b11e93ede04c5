"""The opt-in l1 threshold by Michelot's fixed point (sip_mich.cuh,
SIP_MICH=1; measured slower than the radix rounds on C4, DESIGN.md section
6) against the oracle's Duchi projection: tiny fp64 PARSDMM runs with the
same iteration counts, CG counts and Algorithm-2 branches, and an fp32 run
of the C4 recipe at reduced size within 1e-3."""
import numpy as np
import pytest

import oracle as O
import sip_inputs as G

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1902_09699_b200 import grid_for  # noqa: E402


@pytest.fixture(autouse=True)
def mich_on(monkeypatch):
    monkeypatch.setenv("SIP_MICH", "1")


@pytest.mark.parametrize("seed,shape,kinds", [
    (100, (8, 8), ("bounds", "l1", "slope")),
    (103, (4, 4, 4), ("bounds", "l1", "slope", "dybox")),
    (106, (8, 8), ("bounds", "l1x", "slope")),
    (105, (4, 4, 4), ("bounds", "l1", "cardz", "annulus")),
])
def test_tiny_control_flow_with_michelot(seed, shape, kinds):
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
    np.testing.assert_array_equal(log["branch"][:it], ref.branch[:it])
    assert O.relres(x.cpu().numpy(), ref.x) < 1e-6
    g.close()


def test_c4_recipe_reduced_with_michelot():
    prob = G.c4(shape=(32, 32, 16))
    g = grid_for(prob)
    m = torch.tensor(prob.m, dtype=torch.float32, device="cuda")
    x = torch.empty_like(m)
    g.project(m, x, max_iter=60, tol=1e-3)
    o = dict(prob.options)
    o["max_iter"] = 60
    o["cg_tol_floor"] = 10 * float(np.finfo(np.float32).eps)
    o["decide_f32"] = 1
    ref = O.parsdmm(prob.shape, prob.sets, m.double().cpu().numpy(), **o)
    assert O.relres(x.double().cpu().numpy(), ref.x) < 1e-3
    g.close()
