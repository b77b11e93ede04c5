"""The paper's Fig. 1 experiment on the GPU: PARSDMM (Algorithm
1) against parallel Dykstra with PARSDMM sub-problems (Algorithm 4,
sip_dykstra), counting what the paper counts -- CG iterations
(Dykstra: per outer iteration the largest sub-problem count) and l1-ball
projections -- against the transform-domain feasibility (Eq. 26).

Model: a synthetic 341 x 400 (z, x) geological stand-in (the paper's model
is not in this container): 12 dipping layers U[1500, 4500], two Gaussian
anomalies, N(0, 50^2) noise (seed 7).  Sets as in P:489-491: bounds
[1500, 4500], anisotropic TV l1 ball at 0.4 x ||TV m||_1, D_z x >= 0.
fp32.  Output: profiles/r02_fig1_dykstra.json (+ a printed summary).
usage: python tools/fig1_dykstra.py [--parsdmm-iters 300] [--dykstra-iters 25]
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
import sip_inputs as G  # noqa: E402
from paper_1902_09699_b200 import Grid  # noqa: E402
from sip_inputs import INF, SetDef  # noqa: E402


def model(seed=7, shape=(341, 400)):
    r = np.random.default_rng(seed)
    nz, nx = shape
    zz, xx = np.meshgrid(np.arange(nz), np.arange(nx), indexing="ij")
    depth = zz + np.tan(np.deg2rad(r.uniform(-6, 6))) * (xx - nx / 2)
    edges = np.sort(r.uniform(0, nz, size=11))
    vel = r.uniform(1500, 4500, size=12)
    m = vel[np.searchsorted(edges, depth)]
    for _ in range(2):
        cz, cx, s, a = r.uniform(0, nz), r.uniform(0, nx), r.uniform(15, 40), r.uniform(-600, 600)
        m = m + a * np.exp(-((zz - cz) ** 2 + (xx - cx) ** 2) / (2 * s * s))
    return m + r.normal(0, 50, size=shape)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--parsdmm-iters", type=int, default=300)
    ap.add_argument("--dykstra-iters", type=int, default=25)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_fig1_dykstra.json"))
    a = ap.parse_args()
    shape = (341, 400)
    m = model(shape=shape).astype(np.float32).astype(np.float64)
    sets = [SetDef("I", "bounds", lo=1500.0, hi=4500.0), SetDef("TV", "l1", sigma=0.4, relative=True),
            SetDef("DZ", "bounds", lo=0.0, hi=INF)]
    md = torch.tensor(m, dtype=torch.float32, device="cuda")
    # PARSDMM: the stop test evaluated every iteration, never acted on
    g = Grid(shape, None, "f32")
    for sd in sets:
        g.add_set(sd)
    g.set_option("check_every", 1)
    g.set_option("fixed_work", 1)
    x = torch.empty_like(md)
    t0 = time.time()
    res, _ = g.project(md, x, max_iter=a.parsdmm_iters, tol=1e-3)
    t_p = time.time() - t0
    lg = g.get_log(a.parsdmm_iters)
    n = res["iterations"]
    p_cg = np.cumsum(lg["cg"][:n]).tolist()
    p_l1 = list(range(1, n + 1))                 # one l1-ball projection per iteration
    p_feas = lg["r_feas"][:n].max(axis=1).tolist()
    g.close()
    # parallel Dykstra, PARSDMM sub-problems (the paper's ARADMM role)
    g = Grid(shape, None, "f32")
    for sd in sets:
        g.add_set(sd)
    x2 = torch.empty_like(md)
    t0 = time.time()
    d = g.dykstra(md, x2, max_outer=a.dykstra_iters, tol=0.0, inner_max_iter=200, inner_tol=1e-3)
    t_d = time.time() - t0
    g.close()
    d_cg = np.cumsum(d["cg_max"]).tolist()
    d_l1 = np.cumsum(d["l1_proj"]).tolist()
    d_feas = d["r_feas"].max(axis=1).tolist()

    def first(feas, cost, thr):
        for f, c in zip(feas, cost):
            if f < thr:
                return c
        return None
    summary = {thr: {"parsdmm_cg": first(p_feas, p_cg, thr), "parsdmm_l1": first(p_feas, p_l1, thr),
                     "dykstra_cg": first(d_feas, d_cg, thr), "dykstra_l1": first(d_feas, d_l1, thr)}
               for thr in (1e-1, 3e-2, 1e-2, 3e-3, 1e-3)}
    out = dict(about=__doc__.splitlines()[0], shape=shape, dtype="f32",
               parsdmm=dict(iterations=n, cum_cg=p_cg, cum_l1=p_l1, max_r_feas=p_feas, wall_s=t_p),
               dykstra=dict(iterations=d["iterations"], cum_cg=d_cg, cum_l1=d_l1, max_r_feas=d_feas,
                            inner_iters=d["inner_iters"].tolist(), wall_s=t_d),
               cost_to_reach=summary)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(out, f)
    print("threshold  PARSDMM(CG, l1)  Dykstra(CG, l1)")
    for thr, s in summary.items():
        print(f"{thr:8.0e}  ({s['parsdmm_cg']}, {s['parsdmm_l1']})  ({s['dykstra_cg']}, {s['dykstra_l1']})")
    print(f"final max r_feas: PARSDMM {p_feas[-1]:.2e} after {n} it ({t_p:.2f} s); "
          f"Dykstra {d_feas[-1]:.2e} after {d['iterations']} outer it ({t_d:.2f} s)")


if __name__ == "__main__":
    main()
