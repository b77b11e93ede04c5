"""Algorithm 4 (parallel Dykstra with PARSDMM sub-problems) on the
GPU -- the comparator of the paper's Fig. 1 experiment --
against the oracle's sipref_dykstra: tiny fp64 cases with identical outer
iteration counts and per-iteration counters (largest CG count of the
sub-problems, l1-ball projections, inner iterations per set), x within
1e-8; an fp32 case within 1e-3.  Marked gpu."""
import numpy as np
import pytest

import oracle as O
import sip_inputs as G
from sip_inputs import INF, SetDef

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1902_09699_b200 import Grid  # noqa: E402


def _sets(m):
    return [SetDef("I", "bounds", lo=float(m.min()) + 50.0, hi=float(m.max()) - 50.0),
            SetDef("TV", "l1", sigma=0.5, relative=True),
            SetDef("DZ", "bounds", lo=0.0, hi=INF)]


@pytest.mark.parametrize("shape", [(8, 8), (6, 10), (4, 4, 4)])
def test_dykstra_fp64_matches_oracle(shape):
    m = G.tiny_model(170 + shape[0], shape)
    sets = _sets(m)
    g = Grid(shape, None, "f64")
    for sd in sets:
        g.add_set(sd)
    md = torch.tensor(m, dtype=torch.float64, device="cuda")
    x = torch.empty_like(md)
    d = g.dykstra(md, x, max_outer=12, tol=0.0)
    ref = O.dykstra(shape, sets, m, max_outer=12, tol=0.0)
    assert d["iterations"] == ref["iterations"] == 12
    np.testing.assert_array_equal(d["inner_iters"], ref["inner_iters"])
    np.testing.assert_array_equal(d["cg_max"], ref["cg_max"])
    np.testing.assert_array_equal(d["l1_proj"], ref["l1_proj"])
    assert O.relres(x.cpu().numpy(), ref["x"]) < 1e-8
    np.testing.assert_allclose(d["r_feas"], ref["r_feas"], rtol=1e-6, atol=1e-12)
    g.close()


def test_dykstra_fp32():
    shape = (64, 48)
    m = G.tiny_model(181, shape)
    sets = _sets(m)
    g = Grid(shape, None, "f32")
    for sd in sets:
        g.add_set(sd)
    md = torch.tensor(m.astype(np.float32), device="cuda")
    x = torch.empty_like(md)
    g.dykstra(md, x, max_outer=5, tol=0.0)
    ref = O.dykstra(shape, sets, md.double().cpu().numpy(), max_outer=5, tol=0.0,
                    cg_tol_floor=10 * float(np.finfo(np.float32).eps))
    assert O.relres(x.double().cpu().numpy(), ref["x"]) < 1e-3
    g.close()
