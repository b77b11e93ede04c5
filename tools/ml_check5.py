import sys, copy
import numpy as np
import torch
sys.path.insert(0, ".")
import oracle as O
import sip_inputs as G
from paper_1902_09699_b200 import grid_for
p = G.tiny(125, (16, 8, 16), ("bounds", "l1", "slope"))
q = copy.copy(p); q.shape = (8, 4, 8); q.h = (2.0, 2.0, 2.0); q.m = O.restrict(p.shape, p.m)
xo, sto, logs = O.parsdmm_multilevel(q.shape, q.sets, q.m, 1, h=q.h, **q.options)
g = grid_for(q)
m = torch.tensor(q.m, dtype=torch.float64, device="cuda")
x = torch.empty_like(m)
per, st = g.project_multilevel(m, x, 1, max_iter=200, tol=1e-3)
print([(r["iterations"], r["cg_iterations"]) for r in per], [(lg.iterations, lg.cg_total) for lg in logs])
lg = g.get_log(200); L = logs[0]
np.set_printoptions(precision=12, linewidth=220)
shown = 0
for k in range(200):
    d = np.abs(lg["rho"][k] - L.rho_trace[k]).max() / np.abs(L.rho_trace[k]).max()
    if lg["cg"][k] != L.cg_per_iter[k] or d > 1e-12 or (lg["branch"][k] != L.branch[k]).any():
        print("k", k + 1, "cg", lg["cg"][k], L.cg_per_iter[k], "br", lg["branch"][k], L.branch[k], "drho", d)
        print("   gpu rho", lg["rho"][k], "\n   ora rho", L.rho_trace[k])
        shown += 1
        if shown > 4: break
