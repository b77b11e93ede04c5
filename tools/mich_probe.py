"""Diagnostic: C4 for N natural-mode iterations without graphs, with
SIP_DEBUG_MICH=1 set by the caller (k_mich prints its passes per job)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import sip_inputs as G  # noqa: E402
from paper_1902_09699_b200 import grid_for  # noqa: E402

prob = G.c4()
g = grid_for(prob)
g.set_option("graph_iters", 0)
g.set_option("profile", 1)
m = torch.tensor(prob.m, dtype=torch.float32, device="cuda")
x = torch.empty_like(m)
res, st = g.project(m, x, max_iter=int(sys.argv[1]) if len(sys.argv) > 1 else 20, tol=1e-3)
torch.cuda.synchronize()
print(res["iterations"], {k: v for k, v in g.profile().items() if v[1]})
