"""Parity of the staged z-marching CG kernels (sip_cgs.cuh: bulk-copy plane
tiles with halos in shared memory) with the oracle's CG (Eq. 23, Eq. 25).

The shapes select every tiling the runtime picks: 3D whole-row tiles
(nx = 32 W, 8 rows), 3D 32-chunk tiles with an x halo (nx = 64 W), 2D
whole-row and split-row tiles, ragged z ranges (nz not a multiple of the
CTA's z chunk) and fp64.  The staged kernels are opt-in (SIP_CGS=1: slower than the register-level
kernels on C4, profiles/); the register kernels run the same cases as a
cross-check.  Bar: relative L2 <= 1e-4 (fp32) / 1e-10
(fp64) after 25 CG steps, identical iteration counts.
"""
import numpy as np
import pytest

import oracle as O
from sip_inputs import SetDef

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1902_09699_b200 import Grid  # noqa: E402

TD = {"f32": torch.float32, "f64": torch.float64}

SHAPES = [
    ("f32", (20, 16, 128)),     # whole-row tiles, 8 rows
    ("f32", (37, 16, 128)),     # ragged z chunks
    ("f32", (9, 24, 256)),      # 32-chunk tiles with x halo (nx / W = 64)
    ("f32", (50, 1024)),        # 2D, one tile per row
    ("f32", (33, 2048)),        # 2D, two tiles per row
    ("f64", (12, 16, 64)),      # fp64 whole-row tiles (W = 2)
]


def run(shape, dtype, staged, monkeypatch, eq25=True):
    if staged:
        monkeypatch.setenv("SIP_CGS", "1")
    else:
        monkeypatch.delenv("SIP_CGS", raising=False)
    sets = [SetDef("TV", "l1"), SetDef("DZ", "bounds")]
    g = Grid(shape, None, dtype)
    for sd in sets:
        g.add_set(sd)
    r = np.random.default_rng(5)
    rho = r.uniform(0.1, 3.0, size=len(sets) + 1)
    b = torch.tensor(r.normal(size=shape), dtype=TD[dtype], device="cuda")
    x0 = torch.tensor(r.normal(size=shape), dtype=TD[dtype], device="cuda")
    x = x0.clone()
    it = g.cg(rho, b, x, n_cg=25, eq25=eq25)
    g.close()
    return sets, rho, b.double().cpu().numpy(), x0.double().cpu().numpy(), x.double().cpu().numpy(), it


@pytest.mark.parametrize("eq25", [True, False])
@pytest.mark.parametrize("dtype,shape", SHAPES)
def test_staged_cg_matches_oracle(dtype, shape, eq25, monkeypatch):
    sets, rho, b, x0, x, it = run(shape, dtype, True, monkeypatch, eq25)
    xr, itr, tol, bd = O.cg(shape, sets, rho, b, x0, n_cg=25, eq25=eq25)
    assert it == itr
    assert O.relres(x, xr) <= (1e-4 if dtype == "f32" else 1e-10)


@pytest.mark.parametrize("dtype,shape", SHAPES[:3])
def test_staged_cg_matches_register_kernels(dtype, shape, monkeypatch):
    _, _, _, _, xs, its = run(shape, dtype, True, monkeypatch)
    _, _, _, _, xv, itv = run(shape, dtype, False, monkeypatch)
    assert its == itv
    assert O.relres(xs, xv) <= 1e-5
