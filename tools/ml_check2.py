"""Debug: the level-1 solve of a multilevel run as the finest level of a 2-level run."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import oracle as O
import sip_inputs as G
from paper_1902_09699_b200 import grid_for

def trace(prob, levels):
    xo, sto, logs = O.parsdmm_multilevel(prob.shape, prob.sets, prob.m, levels, h=prob.h, **prob.options)
    # oracle per-iteration traces of the finest level
    g = grid_for(prob)
    m = torch.tensor(prob.m, dtype=torch.float64, device="cuda")
    x = torch.empty_like(m)
    per, st = g.project_multilevel(m, x, levels, max_iter=200, tol=1e-3)
    lg = g.get_log(200)
    L = logs[0]
    n = min(per[0]["iterations"], L.iterations)
    print(prob.name, prob.shape, "levels", levels, "it", per[0]["iterations"], L.iterations)
    for k in range(min(n, 12)):
        print(k + 1, "cg", lg["cg"][k], L.cg_per_iter[k], "rho gpu", np.round(lg["rho"][k], 6), "ora", np.round(L.rho_trace[k], 6))

p = G.tiny(125, (16, 8, 16), ("bounds", "l1", "slope"))
# level 1 of the 3-level run == finest level of a 2-level run on restrict(m)
import copy
p2 = copy.copy(p)
p2.shape = (8, 4, 8)
p2.m = O.restrict(p.shape, p.m)
p2.h = (2.0, 2.0, 2.0)
trace(p2, 2)
q = G.c5(seed=4, shape=(32, 32, 16))
q2 = copy.copy(q); q2.shape = (8, 8, 4); q2.h = (4.0, 4.0, 4.0)
q2.m = O.restrict((16, 16, 8), O.restrict(q.shape, q.m))
q2.dtype = "f64"
trace(q2, 1)
