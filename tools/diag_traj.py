"""Trajectory diagnostics (GPU vs oracle) for the non-convex fp32 configs:
first iteration where the CG count / Alg. 2 branch / cardinality support
differs, and the final relative L2 distance.  Test infrastructure."""
import sys, os, json
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O
import sip_inputs as G
from paper_1902_09699_b200 import grid_for

F32 = float(np.finfo(np.float32).eps)


def first_diff(a, b):
    a = np.asarray(a); b = np.asarray(b)
    n = min(len(a), len(b))
    for i in range(n):
        if not np.array_equal(a[i], b[i]):
            return i + 1
    return None if len(a) == len(b) else n + 1


def single(prob, max_iter, dtype="f32"):
    prob.dtype = dtype
    g = grid_for(prob)
    m = torch.tensor(prob.m, dtype=torch.float32 if dtype == "f32" else torch.float64, device="cuda")
    x = torch.empty_like(m)
    res, st = g.project(m, x, max_iter=max_iter, tol=1e-3)
    lg = g.get_log(max_iter); sup = g.get_support_log(max_iter)
    o = dict(prob.options, max_iter=max_iter)
    if dtype == "f32":
        o["cg_tol_floor"] = 10 * F32
    ref = O.parsdmm(prob.shape, prob.sets, prob.m, **o)
    it = ref.iterations
    out = dict(iters=(res["iterations"], it), rel=O.relres(x.double().cpu().numpy(), ref.x),
               cg=first_diff(lg["cg"][:res["iterations"]], ref.cg_per_iter),
               br=first_diff(lg["branch"][:res["iterations"]], ref.branch),
               supp=first_diff(sup[:res["iterations"]], ref.supp_hash))
    return out


def multi(prob, levels, dtype="f32"):
    prob.dtype = dtype
    g = grid_for(prob)
    m = torch.tensor(prob.m, dtype=torch.float32 if dtype == "f32" else torch.float64, device="cuda")
    x = torch.empty_like(m)
    per, st = g.project_multilevel(m, x, levels, max_iter=200, tol=1e-3)
    o = dict(prob.options)
    if dtype == "f32":
        o["cg_tol_floor"] = 10 * F32
    xo, sto, logs = O.parsdmm_multilevel(prob.shape, prob.sets, prob.m, levels, **o)
    return dict(iters=[(p["iterations"], lg.iterations) for p, lg in zip(per, logs)],
                cg=[(p["cg_iterations"], lg.cg_total) for p, lg in zip(per, logs)],
                rel=O.relres(x.double().cpu().numpy(), xo))


if __name__ == "__main__":
    out = {}
    out["c5s_ml_f32"] = multi(G.c5(seed=4, shape=(32, 32, 16)), 3)
    out["c5s_ml_f64"] = multi(G.c5(seed=4, shape=(32, 32, 16)), 3, "f64")
    out["c5m_ml_f32"] = multi(G.c5(seed=4, shape=(64, 64, 32)), 3)
    for mi in (20, 60, 200):
        out[f"c2_f32_{mi}"] = single(G.c2(), mi)
    print(json.dumps(out, indent=1))
