"""Print the threshold-search jobs of a few iterations (SIP_SEL_DEBUG=1),
select v2 vs the radix rounds (SIP_SEL_V1=1).  Diagnostics."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import sip_inputs as G
from paper_1902_09699_b200 import grid_for
shape = tuple(int(a) for a in sys.argv[1].split("x")) if len(sys.argv) > 1 else (32, 32, 16)
prob = G.c4(shape=shape)
g = grid_for(prob)
g.set_option("graph_iters", 0)
m = torch.tensor(prob.m, dtype=torch.float32, device="cuda")
x = torch.empty_like(m)
g.project(m, x, max_iter=int(os.environ.get("ITERS", "3")), tol=1e-3)
torch.cuda.synchronize()
print("xsum", float(x.double().sum()))
import ctypes
ctypes.CDLL(None).fflush(None)
