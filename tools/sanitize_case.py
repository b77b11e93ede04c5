"""Tiny PARSDMM runs for the guard-band check (SIP_CANARY=1,
tests/test_gpu_canary.py; compute-sanitizer is closed on this pool): every kernel family of the path runs once on small inputs --
vectorised and scalar paths, fp32 and fp64, l1 / cardinality (ties) /
annulus / blur sets, multilevel, virtual z slabs, per-fiber sets.
Test infrastructure."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import sip_inputs as G  # noqa: E402
from paper_1902_09699_b200 import grid_for  # noqa: E402
from sip_inputs import SetDef  # noqa: E402


def run(prob, levels=1, **opts):
    g = grid_for(prob)
    for k, v in opts.items():
        g.set_option(k, v)
    td = torch.float32 if prob.dtype == "f32" else torch.float64
    m = torch.tensor(prob.m, dtype=td, device="cuda")
    x = torch.empty_like(m)
    if levels > 1:
        g.project_multilevel(m, x, levels, max_iter=12, tol=1e-3)
    else:
        g.project(m, x, max_iter=12, tol=1e-3)
    torch.cuda.synchronize()
    g.close()


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    cases = []
    p = G.tiny(101, (8, 8), ("bounds", "l1", "slope", "card", "annulus"))
    cases.append(("tiny_vec_f64", lambda: run(p)))
    cases.append(("tiny_scalar_f64", lambda: run(G.tiny(102, (6, 10), ("bounds", "l1", "slope", "dxbox")))))
    q = G.tiny(105, (8, 8, 16), ("bounds", "l1", "cardz", "annulus"))
    q.dtype = "f32"
    cases.append(("tiny3d_f32", lambda: run(q)))
    cases.append(("tiny3d_f32_graph", lambda: run(q, graph_iters=10, fixed_work=1)))
    cases.append(("blur", lambda: run(G.tiny_blur())))
    r = G.tiny(123, (16, 8, 16), ("bounds", "l1", "slope"))
    cases.append(("multilevel", lambda: run(r, levels=2)))
    cases.append(("slabs", lambda: run(G.tiny(100, (8, 8), ("bounds", "l1", "slope")), virtual_ranks=2)))
    f = G.tiny(106, (8, 16), ("bounds", "slope"))
    f.sets.append(SetDef("DX", "card", k=3, app_mode="x"))
    cases.append(("fibers", lambda: run(f)))
    for name, fn in cases:
        if which in ("all", name):
            fn()
            print("ok", name, flush=True)


if __name__ == "__main__":
    main()
