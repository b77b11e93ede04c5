"""Measurement of the per-fiber path (NEXT-1) on one GPU: the C4 grid
(256 x 256 x 128 fp32, C4's layered model) with C4's bounds and slope sets
plus a per-row cardinality set on D_x (x-fibers, 127 entries, k = half of
each row) and a per-column l1 ball on the model (z-fibers, 256 entries).
Fixed work (50 iterations, stop test evaluated but not acted on).

Prints one JSON line: iterations/s, per-kernel ms per iteration, and the
fiber kernel's achieved bandwidth against its algorithmic bytes:
per launch, each fiber set reads w and writes y and v (3 M words); the
Algorithm-2 products (every other iteration after the first adaptation)
read the previous y and v (2 M), the Eq. 26 check (every 5th iteration)
reads s (1 M): 4.2 M words per set and launch on average.
SIP_FIBER_SORT=1 times the sort kernel instead."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import sip_inputs as G  # noqa: E402
from sip_inputs import SetDef  # noqa: E402
from paper_1902_09699_b200 import grid_for  # noqa: E402


def main():
    shape = (256, 256, 128)
    prob = G.c4()
    sets = [prob.sets[0], prob.sets[2],
            SetDef("DX", "card", k_frac=0.5, relative=True, app_mode="x"),
            SetDef("I", "l1", sigma=2500.0 * shape[0], app_mode="z")]
    p = G.Problem("C4-fibers", shape, "f32", prob.m, sets, options=dict(G.DEFAULT_OPTIONS))
    g = grid_for(p)
    g.set_option("fixed_work", 1)
    m = torch.tensor(p.m, dtype=torch.float32, device="cuda")
    x = torch.empty_like(m)
    iters = 50
    for _ in range(3):
        g.project(m, x, max_iter=iters, tol=1e-3)
    torch.cuda.synchronize()
    ms = []
    for _ in range(5):
        res, st = g.project(m, x, max_iter=iters, tol=1e-3)
        ms.append(res["ms"])
    g.set_option("profile", 1)
    g.project(m, x, max_iter=iters, tol=1e-3)
    prof = g.profile()
    g.set_option("profile", 0)
    M = shape[0] * shape[1] * (shape[2] - 1) + shape[0] * shape[1] * shape[2]
    f_ms, f_n = prof["fiber"]
    bytes_iter = 4.2 * M * 4          # both fiber sets, averaged over the iteration types
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    out = dict(workload="C4 grid + per-row card(D_x) + per-column l1 (fp32), 50 fixed iterations",
               path="sort" if os.environ.get("SIP_FIBER_SORT") else "warp",
               it_per_s=iters / (min(ms) / 1e3),
               ms_per_iter={k: v[0] / iters for k, v in prof.items() if v[1]},
               fiber_launches=f_n,
               fiber_us_per_launch=1e3 * f_ms / max(f_n, 1),
               fiber_us_per_iter=1e3 * f_ms / iters,
               fiber_GBps=bytes_iter / (f_ms / iters / 1e3) / 1e9 if f_ms else None,
               peaks=peaks)
    print(json.dumps(out), flush=True)
    g.close()


if __name__ == "__main__":
    main()
