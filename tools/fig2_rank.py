"""The paper's Fig. 2 experiment on the GPU: a non-convex
intersection -- bounds and a rank constraint on the vertical gradient,
{m : rank(D_z m) <= r} (the (n_z - 1) x n_x matrix view, reading L29)
-- projected by PARSDMM (Algorithm 1, single level as in P:520) and by
parallel Dykstra with PARSDMM sub-problems (Algorithm 4, sip_dykstra).
Counted as the paper counts: CG iterations (Dykstra: per outer
iteration the largest sub-problem count) and projections onto the rank set
(each an SVD; PARSDMM: one per iteration, the Eq. 26 evaluation not
counted; Dykstra: the rank sub-problem's inner iterations), against the
largest Eq. 26 feasibility.

Model: the 341 x 400 stand-in of tools/fig1_dykstra.py (seed 7), fp32; sets
bounds [1500, 4500] and rank(D_z x) <= r (default r = 8).
Output: profiles/r02_fig2_rank.json (+ a printed summary).
usage: python tools/fig2_rank.py [--rank 8] [--parsdmm-iters 300] [--dykstra-iters 10]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from fig1_dykstra import model  # noqa: E402
from paper_1902_09699_b200 import Grid  # noqa: E402
from sip_inputs import SetDef  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rank", type=int, default=8)
    ap.add_argument("--parsdmm-iters", type=int, default=300)
    ap.add_argument("--dykstra-iters", type=int, default=10)
    ap.add_argument("--inner-iters", type=int, default=100)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_fig2_rank.json"))
    a = ap.parse_args()
    shape = (341, 400)
    m = model(shape=shape).astype(np.float32).astype(np.float64)
    sets = [SetDef("I", "bounds", lo=1500.0, hi=4500.0), SetDef("DZ", "rank", k=a.rank)]
    md = torch.tensor(m, dtype=torch.float32, device="cuda")
    g = Grid(shape, None, "f32")
    for sd in sets:
        g.add_set(sd)
    g.set_option("check_every", 1)
    g.set_option("fixed_work", 1)
    x = torch.empty_like(md)
    torch.cuda.synchronize()
    t0 = time.time()
    res, _ = g.project(md, x, max_iter=a.parsdmm_iters, tol=1e-3)
    torch.cuda.synchronize()
    t_p = time.time() - t0
    lg = g.get_log(a.parsdmm_iters)
    n = res["iterations"]
    p_cg = np.cumsum(lg["cg"][:n]).tolist()
    p_svd = list(range(1, n + 1))
    p_feas = lg["r_feas"][:n].max(axis=1).tolist()
    p_feas_sets = lg["r_feas"][:n].tolist()
    g.close()
    g = Grid(shape, None, "f32")
    for sd in sets:
        g.add_set(sd)
    x2 = torch.empty_like(md)
    t0 = time.time()
    d = g.dykstra(md, x2, max_outer=a.dykstra_iters, tol=0.0, inner_max_iter=a.inner_iters, inner_tol=1e-3)
    torch.cuda.synchronize()
    t_d = time.time() - t0
    g.close()
    d_cg = np.cumsum(d["cg_max"]).tolist()
    d_svd = np.cumsum(d["inner_iters"][:, 1]).tolist()
    d_feas = d["r_feas"].max(axis=1).tolist()

    def first(feas, cost, thr):
        for f, c in zip(feas, cost):
            if f < thr:
                return c
        return None
    summary = {thr: {"parsdmm_cg": first(p_feas, p_cg, thr), "parsdmm_svd": first(p_feas, p_svd, thr),
                     "dykstra_cg": first(d_feas, d_cg, thr), "dykstra_svd": first(d_feas, d_svd, thr)}
               for thr in (1e-1, 3e-2, 1e-2, 3e-3, 1e-3)}
    out = dict(about=__doc__.splitlines()[0], shape=shape, dtype="f32", rank=a.rank,
               parsdmm=dict(iterations=n, cum_cg=p_cg, cum_svd=p_svd, max_r_feas=p_feas, r_feas=p_feas_sets,
                            wall_s=t_p),
               dykstra=dict(iterations=d["iterations"], cum_cg=d_cg, cum_svd=d_svd, max_r_feas=d_feas,
                            r_feas=d["r_feas"].tolist(), inner_iters=d["inner_iters"].tolist(), wall_s=t_d),
               cost_to_reach=summary)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(out, f)
    print("threshold  PARSDMM(CG, SVD)  Dykstra(CG, SVD)")
    for thr, s in summary.items():
        print(f"{thr:8.0e}  ({s['parsdmm_cg']}, {s['parsdmm_svd']})  ({s['dykstra_cg']}, {s['dykstra_svd']})")
    print(f"final r_feas (bounds, rank): PARSDMM {p_feas_sets[-1]} after {n} it ({t_p:.2f} s); "
          f"Dykstra {d['r_feas'][-1].tolist()} after {d['iterations']} outer it ({t_d:.2f} s)")


if __name__ == "__main__":
    main()
