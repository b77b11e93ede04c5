"""Debug helper: GPU (f32 and f64) vs oracle on a config, with trajectories."""
import sys
import time
import numpy as np
import torch
sys.path.insert(0, ".")
import oracle as O
import sip_inputs as G
from paper_1902_09699_b200 import grid_for

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
max_iter = int(sys.argv[2]) if len(sys.argv) > 2 else 200
prob = G.CONFIGS[name]()
t = time.time()
ref = O.parsdmm(prob.shape, prob.sets, prob.m, max_iter=max_iter, n_cg=10, rho0=1e-2,
                cg_tol_floor=10 * float(np.finfo(np.float32).eps))
print(f"oracle {time.time()-t:.1f}s it={ref.iterations} conv={ref.converged} cg={ref.cg_total} "
      f"feas={ref.r_feas} evol={ref.r_evol:.3e}")
for dt in ("f32", "f64"):
    prob.dtype = dt
    g = grid_for(prob)
    td = torch.float32 if dt == "f32" else torch.float64
    m = torch.tensor(prob.m, dtype=td, device="cuda")
    x = torch.empty_like(m)
    res, st = g.project(m, x, max_iter=max_iter)
    lg = g.get_log(max_iter)
    xr = x.double().cpu().numpy().ravel()
    print(f"gpu {dt} ms={res['ms']:.1f} it={res['iterations']} conv={res['converged']} cg={res['cg_iterations']} "
          f"feas={res['r_feas']} evol={res['r_evol']:.3e} rel={O.relres(xr, ref.x):.3e}")
    k = min(res["iterations"], ref.iterations)
    diff = np.nonzero(lg["cg"][:k] != ref.cg_per_iter[:k])[0]
    print("  first cg-count difference at k =", diff[:5] + 1 if len(diff) else None)
    dr = np.abs(lg["rho"][:k] - ref.rho_trace[:k]) / np.abs(ref.rho_trace[:k])
    bad = np.nonzero(dr.max(axis=1) > 1e-3)[0]
    print("  first rho divergence > 1e-3 at k =", bad[:3] + 1 if len(bad) else None)
    g.close()
