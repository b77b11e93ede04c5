"""Debug helper: first iteration where GPU and oracle traces diverge."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import oracle as O
import sip_inputs as G
from paper_1902_09699_b200 import grid_for

def main(seed, shape, kinds, max_iter=200):
    prob = G.tiny(seed, shape, kinds)
    g = grid_for(prob)
    m = torch.tensor(prob.m, dtype=torch.float64, device="cuda")
    x = torch.empty_like(m)
    res, st = g.project(m, x, max_iter=max_iter)
    lg = g.get_log(max_iter)
    ref = O.parsdmm(prob.shape, prob.sets, prob.m, max_iter=max_iter, n_cg=10, rho0=1e-2)
    n = min(res["iterations"], ref.iterations)
    print("iters gpu", res["iterations"], "oracle", ref.iterations)
    for k in range(n):
        dr = np.abs(lg["rho"][k] - ref.rho_trace[k]) / np.abs(ref.rho_trace[k])
        line = f"k={k+1} cg {lg['cg'][k]}/{ref.cg_per_iter[k]} br {lg['branch'][k]}/{ref.branch[k]} drho {dr.max():.2e}"
        if not np.isnan(ref.r_evol_trace[k]):
            line += f" evol {lg['r_evol'][k]:.6e}/{ref.r_evol_trace[k]:.6e} feas {lg['r_feas'][k]}/{ref.r_feas_trace[k]}"
        print(line)


def detail(seed, shape, kinds, k0, k1, max_iter=200):
    prob = G.tiny(seed, shape, kinds)
    g = grid_for(prob)
    m = torch.tensor(prob.m, dtype=torch.float64, device="cuda")
    x = torch.empty_like(m)
    res, st = g.project(m, x, max_iter=max_iter)
    lg = g.get_log(max_iter)
    ref = O.parsdmm(prob.shape, prob.sets, prob.m, max_iter=max_iter, n_cg=10, rho0=1e-2)
    np.set_printoptions(precision=10, linewidth=200)
    for k in range(k0 - 1, k1):
        print(k + 1, "gpu rho", lg["rho"][k], "gam", lg["gamma"][k], lg["branch"][k])
        print(k + 1, "ora rho", ref.rho_trace[k], "gam", ref.gamma_trace[k], ref.branch[k])

if __name__ == "__main__":
    detail(101, (8, 8), ("bounds", "l1", "slope", "card", "annulus"), 70, 82)
