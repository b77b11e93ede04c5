"""Run the CPU oracle ONCE on a full-size BASELINE.json configuration and store
what the GPU parity tests compare against (tests/golden/fullsize_<cfg>.json).

Test infrastructure: this script calls only ``oracle/`` (fp64, single thread)
and the seeded input generators ``sip_inputs``; nothing here comes from the
CUDA path.  SURVEY.md 8(c)/8(d): "full C4/C5 runs done once, for parity only".

Natural mode (Eq. 25 on, stop test acted on, max 200 iterations per level,
reading L11); fp32 configurations take the Eq. 25 floor 10*FLT_EPSILON
(reading L18).  The oracle gets the fp32-rounded m, the same bits the GPU gets.

Stored per level: iteration count, converged flag, CG count per iteration,
Alg. 2 branch per iteration and set, rho / gamma traces, Eq. 26 / Eq. 27
traces, the cardinality support fingerprint per iteration, final r_feas /
r_evol; at the finest level also ||x||, sha256 of x (fp64 bytes) and a strided
subsample of x (every `stride`-th point).

usage: python tools/oracle_fullsize.py C4|C5 [--out tests/golden]
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
import sip_inputs as G  # noqa: E402

F32_EPS = float(np.finfo(np.float32).eps)
N_SUB = 16384


def _clean(a):
    """JSON-safe list (NaN -> None)"""
    a = np.asarray(a)
    if a.dtype.kind == "f":
        return [None if not np.isfinite(v) else float(v) for v in a.ravel()]
    return [int(v) for v in a.ravel()]


def level_record(r):
    return dict(
        iterations=int(r.iterations), converged=bool(r.converged), cg_total=int(r.cg_total),
        cg_per_iter=_clean(r.cg_per_iter), branch=np.asarray(r.branch).tolist(),
        rho_trace=np.asarray(r.rho_trace).tolist(), gamma_trace=np.asarray(r.gamma_trace).tolist(),
        r_feas_trace=[[None if not np.isfinite(v) else float(v) for v in row] for row in r.r_feas_trace],
        r_evol_trace=_clean(r.r_evol_trace),
        supp_hash=[[str(int(v)) for v in row] for row in r.supp_hash],
        r_feas=_clean(r.r_feas), r_evol=float(r.r_evol),
        rho=_clean(r.rho), gamma=_clean(r.gamma),
    )


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfg", choices=["C4", "C5"])
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden"))
    ap.add_argument("--max-iter", type=int, default=200)
    a = ap.parse_args()
    prob = G.c4() if a.cfg == "C4" else G.c5()
    m = prob.m.astype(np.float32).astype(np.float64) if prob.dtype == "f32" else prob.m
    opts = dict(prob.options)
    opts["max_iter"] = a.max_iter
    if prob.dtype == "f32":
        opts["cg_tol_floor"] = 10 * F32_EPS
    t0 = time.time()
    if prob.n_levels > 1:
        x, st, logs = O.parsdmm_multilevel(prob.shape, prob.sets, m, prob.n_levels, **opts)
        levels = [level_record(r) for r in logs]
    else:
        r = O.parsdmm(prob.shape, prob.sets, m, **opts)
        x, levels = r.x, [level_record(r)]
    wall = time.time() - t0
    x = np.ascontiguousarray(x, dtype=np.float64).ravel()
    stride = max(1, x.size // N_SUB)
    rec = dict(
        about=("Oracle (oracle/sipref.c, fp64, 1 thread) on full-size " + a.cfg +
               ", natural mode; written by tools/oracle_fullsize.py (calls only oracle/ "
               "and sip_inputs). SURVEY.md 8(c)/8(d)."),
        cfg=a.cfg, shape=list(prob.shape), dtype=prob.dtype, n_levels=prob.n_levels,
        sets=[f"{s.op}:{s.kind}" for s in prob.sets], options=opts,
        levels=levels,   # level 0 = finest
        x_norm=float(np.linalg.norm(x)), x_sha256=hashlib.sha256(x.tobytes()).hexdigest(),
        stride=stride, x_sub=[float(v) for v in x[::stride]],
        wall_s=wall, host_cpu=_cpu_model(),
    )
    os.makedirs(a.out, exist_ok=True)
    path = os.path.join(a.out, f"fullsize_{a.cfg}.json")
    with open(path, "w") as f:
        json.dump(rec, f)
    print(path, "iterations", [lv["iterations"] for lv in levels], "wall", round(wall, 1), "s")


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


if __name__ == "__main__":
    main()
