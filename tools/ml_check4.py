import sys, copy
import numpy as np
import torch
sys.path.insert(0, ".")
import oracle as O
import sip_inputs as G
from paper_1902_09699_b200 import grid_for
p = G.tiny(125, (16, 8, 16), ("bounds", "l1", "slope"))
for levels in (1, 2, 3):
    xo, sto, logs = O.parsdmm_multilevel(p.shape, p.sets, p.m, levels, **p.options)
    g = grid_for(p)
    m = torch.tensor(p.m, dtype=torch.float64, device="cuda")
    x = torch.empty_like(m)
    per, st = g.project_multilevel(m, x, levels, max_iter=200, tol=1e-3)
    print(levels, [(q["iterations"], q["cg_iterations"]) for q in per], [(lg.iterations, lg.cg_total) for lg in logs],
          O.relres(x.cpu().numpy(), xo))
    if levels == 2:
        lg = g.get_log(200); L = logs[0]
        for k in range(200):
            if lg["cg"][k] != L.cg_per_iter[k] or np.abs(lg["rho"][k] - L.rho_trace[k]).max() > 1e-9 * np.abs(L.rho_trace[k]).max():
                print("first diff at k", k + 1, lg["cg"][k], L.cg_per_iter[k], lg["rho"][k], L.rho_trace[k], lg["branch"][k], L.branch[k])
                break
