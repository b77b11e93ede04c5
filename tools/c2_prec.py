import sys, copy, time
import numpy as np
import torch
sys.path.insert(0, ".")
import oracle as O
import sip_inputs as G
from paper_1902_09699_b200 import grid_for
base = G.c2()
def run(prob, iters, tag):
    t = time.time()
    ref = O.parsdmm(prob.shape, prob.sets, prob.m, max_iter=iters, n_cg=10, rho0=1e-2,
                    cg_tol_floor=10 * float(np.finfo(np.float32).eps))
    g = grid_for(prob)
    m = torch.tensor(prob.m, dtype=torch.float32, device="cuda")
    x = torch.empty_like(m)
    res, st = g.project(m, x, max_iter=iters)
    print(f"{tag} iters={iters} rel={O.relres(x.double().cpu().numpy(), ref.x):.3e} "
          f"it={res['iterations']}/{ref.iterations} conv={res['converged']}/{ref.converged} ({time.time()-t:.0f}s)", flush=True)
for iters in (20, 60):
    run(base, iters, "C2 full")
nocard = copy.copy(base); nocard.sets = [s for s in base.sets if s.kind != "card"]
run(nocard, 60, "C2 no-card")
