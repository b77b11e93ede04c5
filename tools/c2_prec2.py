import sys, copy, time
import numpy as np
import torch
sys.path.insert(0, ".")
import oracle as O
import sip_inputs as G
from paper_1902_09699_b200 import grid_for
base = G.c2()
for iters in (60, 200):
    t = time.time()
    ref = O.parsdmm(base.shape, base.sets, base.m, max_iter=iters, n_cg=10, rho0=1e-2, decide_f32=1,
                    cg_tol_floor=10 * float(np.finfo(np.float32).eps))
    g = grid_for(base)
    m = torch.tensor(base.m, dtype=torch.float32, device="cuda")
    x = torch.empty_like(m)
    res, st = g.project(m, x, max_iter=iters)
    print(f"decide_f32 iters={iters} rel={O.relres(x.double().cpu().numpy(), ref.x):.3e} ({time.time()-t:.0f}s)", flush=True)
