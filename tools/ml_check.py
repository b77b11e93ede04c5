"""Debug helper: multilevel GPU vs oracle per level."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import oracle as O
import sip_inputs as G
from paper_1902_09699_b200 import grid_for

def run(prob, levels, dt):
    prob.dtype = dt
    o = dict(prob.options)
    if dt == "f32":
        o["cg_tol_floor"] = 10 * float(np.finfo(np.float32).eps)
    xo, sto, logs = O.parsdmm_multilevel(prob.shape, prob.sets, prob.m, levels, **o)
    g = grid_for(prob)
    m = torch.tensor(prob.m, dtype=torch.float32 if dt == "f32" else torch.float64, device="cuda")
    x = torch.empty_like(m)
    per, st = g.project_multilevel(m, x, levels, max_iter=200, tol=1e-3)
    print(prob.name, prob.shape, dt, "rel", O.relres(x.double().cpu().numpy(), xo))
    for l in range(levels):
        print(f"  level {l}: gpu it={per[l]['iterations']} cg={per[l]['cg_iterations']} conv={per[l]['converged']}"
              f" | oracle it={logs[l].iterations} cg={logs[l].cg_total} conv={logs[l].converged}")
        print("     gpu rho", np.round(per[l]["rho"], 6), "ora rho", np.round(logs[l].rho, 6))

run(G.tiny(125, (16, 8, 16), ("bounds", "l1", "slope")), 3, "f64")
run(G.tiny(122, (16, 16), ("bounds", "l1", "slope")), 2, "f64")
run(G.c5(seed=4, shape=(32, 32, 16)), 3, "f64")
run(G.c5(seed=4, shape=(32, 32, 16)), 3, "f32")
