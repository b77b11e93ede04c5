import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import oracle as O
from sip_inputs import SetDef
from paper_1902_09699_b200 import Grid
for shape, w in [((4, 4), np.diag([3.0, 2.0, 1.0, 0.5]).ravel()), ((6, 8), np.random.default_rng(0).normal(size=48))]:
    sd = SetDef("I", "rank", k=2)
    g = Grid(shape, None, "f64"); g.add_set(sd)
    m = torch.zeros(shape, dtype=torch.float64, device="cuda"); x = torch.empty_like(m)
    g.project(m, x, max_iter=1)
    wd = torch.tensor(w, dtype=torch.float64, device="cuda"); y = torch.empty_like(wd)
    g.project_set(0, wd, y)
    print(shape, "gpu", np.round(y.cpu().numpy(), 4)[:16])
    print(shape, "ref", np.round(O.project(sd, w, shape=shape), 4)[:16])
