import sys, copy
import numpy as np
import torch
sys.path.insert(0, ".")
import oracle as O
import sip_inputs as G
from paper_1902_09699_b200 import grid_for
q = G.c5(seed=4, shape=(32, 32, 16)); q.dtype = "f64"
for levels in (1, 2, 3):
    xo, sto, logs = O.parsdmm_multilevel(q.shape, q.sets, q.m, levels, **q.options)
    g = grid_for(q)
    m = torch.tensor(q.m, dtype=torch.float64, device="cuda")
    x = torch.empty_like(m)
    per, st = g.project_multilevel(m, x, levels, max_iter=200, tol=1e-3)
    print(levels, [p["iterations"] for p in per], [lg.iterations for lg in logs],
          O.relres(x.cpu().numpy(), xo))
# 2-level on the half grid with CPU restriction
q2 = copy.copy(q); q2.shape = (16, 16, 8); q2.h = (2.0, 2.0, 2.0); q2.m = O.restrict(q.shape, q.m)
xo, sto, logs = O.parsdmm_multilevel(q2.shape, q2.sets, q2.m, 2, h=q2.h, **q2.options)
g = grid_for(q2)
m = torch.tensor(q2.m, dtype=torch.float64, device="cuda")
x = torch.empty_like(m)
per, st = g.project_multilevel(m, x, 2, max_iter=200, tol=1e-3)
print("half", [p["iterations"] for p in per], [lg.iterations for lg in logs], O.relres(x.cpu().numpy(), xo))
