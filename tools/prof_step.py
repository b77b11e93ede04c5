"""One fixed-work projection of a config (for ncu launch lists / captures)."""
import argparse
import sys
import torch
sys.path.insert(0, ".")
import sip_inputs as G
from paper_1902_09699_b200 import grid_for

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C4")
ap.add_argument("--iters", type=int, default=2)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--graph", type=int, default=5)
a = ap.parse_args()
prob = G.CONFIGS[a.config]()
g = grid_for(prob)
g.set_option("fixed_work", 1)
g.set_option("eq25", 0)
g.set_option("graph_iters", a.graph)
dt = torch.float32 if prob.dtype == "f32" else torch.float64
m = torch.tensor(prob.m, dtype=dt, device="cuda")
x = torch.empty_like(m)
for _ in range(a.reps):
    res, st = g.project(m, x, max_iter=a.iters)
torch.cuda.synchronize()
print("ok", res["ms"], g.launch_count())
