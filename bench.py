"""Benchmark of the B200 PARSDMM hot path (arXiv 1902.09699).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4]
                    [--iters-per-step 10] [--impl cuda|reference]

A step is one call of the public API, sip_project, in fixed-work mode
(Eq. 25 off -> exactly n_cg = 10 CG steps per iteration; the
Eq. 26-28 stop test computed but not acted on; Algorithm 2 on) running
`iters_per_step` outer PARSDMM iterations on the config's seeded synthetic
model.  Ten iterations cover every row of SURVEY 8(a): rhs, CG, transform +
relaxation, pointwise / l1 / cardinality / annulus projections, duals,
5 adapt calls and 2 stop checks.  The metric is BASELINE.json's:
PARSDMM iterations/s (also grid-points x sets / s and the HBM roofline).

value   = iterations of all ranks / max over ranks of the summed device time
          of the K timed steps (library CUDA events around each call; L2 is
          flushed by a 256 MiB write between steps, outside the timing).
e2e     = the same metric through the same call with host (pinned) m and x:
          the H2D copy of m and the D2H copy of x are inside the timed call.
roofline: the dominant kernel (k_cg2: x += a p, r -= a C p) -- its device
          time comes from CUDA event nodes captured in the iteration graph
          (option "profile") in a separate profiled step of the same workload.
--impl reference: the CPU oracle (oracle/, plain C fp64, 1 thread) timed on
          a bounded sample of the same workload (the reference arm of this
          tier: there is no reference implementation).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import sip_inputs as G  # noqa: E402

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    return PEAKS_FALLBACK


def op_len(shape, op):
    """compact length M of an operator (for the algorithmic byte model)"""
    if len(shape) == 2:
        nz, nx = shape
        ny = 1
    else:
        nz, ny, nx = shape
    N = nz * ny * nx
    dz, dy, dx = (nz - 1) * ny * nx, (nz * (ny - 1) * nx if len(shape) == 3 else 0), nz * ny * (nx - 1)
    return {"I": N, "DZ": dz, "DY": dy, "DX": dx, "TV": dz + dy + dx}.get(op, N // 2)


def byte_model(prob, n_cg=10, word=4):
    """algorithmic bytes (with the CG's x update deferred to one
    pass after the loop: DESIGN.md section 6): per CG kernel launch and per
    iteration"""
    N = prob.N
    Ms = [op_len(prob.shape, sd.op) for sd in prob.sets] + [N]
    SM = sum(Ms)
    T = sum(op_len(prob.shape, sd.op) for sd in prob.sets if sd.kind in ("l1", "card", "annulus", "l2"))
    cg1 = 3 * N * word          # read r, p_{j-1}; write p_j
    cg2 = 3 * N * word          # read r, p_j; write r (x is not touched inside the loop)
    cgx = (n_cg + 2) * N * word  # x += sum_j alpha_j p_j: read x and the n_cg p_j; write x
    a, c = 0.5, 0.2
    it = word * (6 * N * n_cg + (n_cg + 2) * N + (2 * SM + 2 * N) + (4 * SM + 2 * N) + T + N
                 + a * (4 * SM + 2 * N) + c * (5 * N + T))
    return dict(cg1=cg1, cg2=cg2, cgx=cgx, iteration=it)


def kernel_bytes(prob, k, n_cg=10, word=4):
    """algorithmic bytes of every kernel kind in PARSDMM iteration k (1-based;
    adapt when k is odd with Alg. 2 products from k = 3 on, check when
    k % 5 == 0): the minimum each kind must move -- every operand read once,
    every result written once, neighbours of a stencil from on-chip reuse
    (DESIGN.md section 6).  Compact lengths M_i (shared sizes)."""
    N = prob.N
    sets = prob.sets
    M = [op_len(prob.shape, sd.op) for sd in sets] + [N]               # + distance block
    point = [i for i, sd in enumerate(sets) if sd.kind == "bounds"] + [len(sets)]
    glob = [i for i, sd in enumerate(sets) if sd.kind in ("l1", "card", "annulus", "l2")]
    radix = [i for i, sd in enumerate(sets) if sd.kind in ("l1", "card") and not sd.app_mode]
    SM, SMp = sum(M), sum(M[i] for i in point)
    T, Tr = sum(M[i] for i in glob), sum(M[i] for i in radix)
    adapt, dots, check = k % 2 == 1, k % 2 == 1 and k >= 3, k % 5 == 0
    # full reads of w per radix job: fp32 (select v2, sip_select2.cuh) one
    # streaming pass -- round A runs inside pass 1, the candidate rounds read
    # only the candidates; fp64 radix rounds read w in each of their 6 rounds
    rounds = 1 if word == 4 else 6
    by = {
        "rhs": 2 * SM + 2 * N,                               # y_i, v_i, x -> r
        "cg1": 3 * N * n_cg, "cg2": 3 * N * n_cg,
        "cgx": (n_cg + 2) * N,
        "pass1": (N + N + N + 2 * SM + 2 * SMp + T           # x, m, history write; y, v; y, v (pointwise); w
                  + (SM if adapt else 0)                     # v_hat write
                  + ((SM + 2 * N + 2 * SMp) if dots else 0)  # v_hat^{k0}, x^{k0} r/w, y^{k0} v^{k0} (pointwise)
                  + ((Tr + 5 * N) if check else 0)),         # s of l1/card sets, 5 history vectors
        "select": rounds * Tr * (2 if check else 1),         # w (and s on check iterations)
        "pass2": 3 * T + (2 * T if dots else 0) + (Tr if check else 0),
    }
    return {kk: v * word for kk, v in by.items()}
class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region"""

    def __init__(self, gpu=0):
        self.gpu, self.rows, self.proc = gpu, [], None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([s.strip() for s in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm = [float(r[0]) for r in self.rows if r and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 3 + i and r[3 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def max_over_ranks(v, world, device=None):
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(v, world, device=None):
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device=device)
    dist.all_reduce(t)
    return float(t.item())


def workload_config(prob, args, world=None):
    """the `config` object of both arms (same workload, same keys)"""
    world = world if world is not None else args.gpus
    return {"workload": f"{prob.name} {'x'.join(map(str, prob.shape))} "
                        f"{', '.join(sd.op + ':' + sd.kind for sd in prob.sets)}",
            "grid": list(prob.shape), "sets": len(prob.sets), "iters_per_step": args.iters_per_step,
            "levels": prob.n_levels if getattr(args, "multilevel", False) else 1,
            "n_cg": args.n_cg, "mode": "fixed_work (Eq.25 off, stop test not acted on)",
            "l2": "flushed (256 MiB write) between timed steps",
            "parallelism": ("1 GPU" if world == 1 else f"z-slab x{world} (NCCL halos + gathered reductions)")
                           + (f", {args.virtual_ranks} virtual z-slabs on the GPU" if args.virtual_ranks > 1 else "")}


# ------------------------------------------------------------------ oracle arm
def oracle_sample(prob, iters, reps=1):
    """the CPU oracle (fixed-work PARSDMM) on the same workload; seconds/iteration"""
    import oracle as O
    opts = dict(prob.options)
    opts.update(max_iter=iters, eq25=0, fixed_work=1)
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        O.parsdmm(prob.shape, prob.sets, prob.m, **opts)
        ts.append(time.perf_counter() - t0)
    return ts


def run_reference(args, prob):
    world, rank, _ = dist_init()
    if rank != 0:
        return 0
    ips = args.ref_iters
    # warm-up steps (untimed): the plain C oracle has no JIT or caches to warm;
    # a small case keeps the whole --steps K --warmup W run within minutes
    small = G.tiny(100, (8, 8), ("bounds", "l1", "slope"))
    for _ in range(args.warmup):
        oracle_sample(small, 1)
    ts = []
    for _ in range(args.steps):
        ts += oracle_sample(prob, ips)
    total = sum(ts)
    val = args.steps * ips / total
    line = {
        "impl": "reference", "metric": "PARSDMM iterations/s", "value": val, "unit": "it/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(prob, args),
        "pts_sets_per_s": val * prob.N * len(prob.sets),
        "cpu_baseline": {"value": val, "unit": "it/s", "cores": 1, "kind": "oracle",
                         "sample": f"{args.steps} steps x {ips} fixed-work iterations of {prob.name} "
                                   f"(single-threaded fp64 C oracle)", **host_info()},
        "e2e": {"value": val, "unit": "it/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ CUDA arm
KINDS_RL = ("rhs", "cg1", "cg2", "cgx", "pass1", "select", "pass2")
KNAME = {"rhs": "k_rhsp", "cg1": "k_cg1f", "cg2": "k_cg2f", "cgx": "k_cgx", "pass1": "k_pass1t",
         "select": "k_selectf", "pass2": "k_pass2t"}


def host_info():
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


def roofline_table(prob, prof, ips, n_cg, word, peak, level_shapes=None):
    """per kernel kind: algorithmic bytes of the profiled step / its device
    time (CUDA event nodes in the graph) against the measured copy peak"""
    tot = {k: 0.0 for k in KINDS_RL}
    probs = [prob] if level_shapes is None else level_shapes
    for pb in probs:
        for k in range(1, ips + 1):
            for kk, v in kernel_bytes(pb, k, n_cg, word).items():
                tot[kk] += v
    out = {}
    for kk in KINDS_RL:
        ms, n = prof.get(kk, (0.0, 0))
        if ms <= 0 or n == 0:
            continue
        gbs = tot[kk] / (ms / 1e3) / 1e9
        out[kk] = {"kernel": KNAME[kk], "ms_per_step": ms, "launches": n,
                   "bytes_per_step": tot[kk], "achieved_gbs": gbs, "frac": gbs / peak}
    return out


def run_cuda(args, prob):
    import torch
    world, rank, local = dist_init()
    torch.cuda.set_device(local)
    from paper_1902_09699_b200 import grid_for
    from paper_1902_09699_b200.dist import comm_desc, local_slab_of

    comm = None
    m_np = prob.m
    if world > 1:
        # z slabs over NCCL: strong scaling of one problem;
        # torch.distributed only bootstraps the library's NCCL communicator
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        comm = comm_desc()
        m_np = local_slab_of(prob.m, world, rank)
    dt = torch.float32 if prob.dtype == "f32" else torch.float64
    word = 4 if prob.dtype == "f32" else 8
    ips = args.iters_per_step
    levels = prob.n_levels if args.multilevel else 1
    g = grid_for(prob, comm=comm)
    g.set_option("fixed_work", 1)
    g.set_option("eq25", 0)
    g.set_option("n_cg", args.n_cg)
    if args.virtual_ranks > 1:
        g.set_option("virtual_ranks", args.virtual_ranks)
    m = torch.tensor(m_np, dtype=dt, device="cuda").contiguous()
    x = torch.empty_like(m)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")   # 256 MiB > L2

    def call(mm, xx):
        if levels > 1:
            per, st = g.project_multilevel(mm, xx, levels, max_iter=ips, tol=1e-3)
            return sum(p["ms"] for p in per), per
        res, st = g.project(mm, xx, max_iter=ips, tol=1e-3)
        return res["ms"], [res]

    for _ in range(args.warmup):
        call(m, x)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    times, launches, lvl_ms = [], 0, [0.0] * levels
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            ms, per = call(m, x)
            times.append(ms)
            for l, p in enumerate(per):
                lvl_ms[l] += p["ms"]
            launches += g.launch_count()
        torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    t_total = max_over_ranks(sum(times), world, "cuda")          # ms, slowest rank
    its_per_step = ips * levels
    value_job = args.steps * its_per_step / (t_total / 1e3)      # iterations of the one (sharded) problem

    # e2e: host pinned m / x, copies inside the timed call
    mh = torch.tensor(m_np, dtype=dt).pin_memory()
    xh = torch.empty_like(mh).pin_memory()
    call(mh, xh)
    etimes = []
    for _ in range(max(1, args.steps // 2)):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        call(mh, xh)
        etimes.append(time.perf_counter() - t0)
    e2e_t = max_over_ranks(sum(etimes), world, "cuda")
    e2e_val = len(etimes) * its_per_step / e2e_t
    nbytes = m_np.size * word                                     # this rank's slab (one GPU: the grid)

    # profiled step: per-kernel device time from event nodes in the graph
    g.set_option("profile", 1)
    flush.zero_()
    torch.cuda.synchronize()
    call(m, x)
    prof = g.profile()
    g.set_option("profile", 0)
    peaks = load_peaks()
    lv_probs = None
    if levels > 1:   # the profile is the finest level's (the library profiles the last engine)
        lv_probs = [prob]
    scale = m_np.size / prob.N                                    # this rank's share of the bytes
    table = roofline_table(prob, prof, ips, args.n_cg, word, peaks["hbm_gbs"], lv_probs)
    if "select" in table and world == 1:   # the single-rank threshold searches
        table["select"]["kernel"] = ("k_selsmall" if 3 * prob.N <= 8192 else
                                     "k_selB+k_selC" if word == 4 else "k_selectf")
    for v in table.values():
        v["bytes_per_step"] *= scale
        v["achieved_gbs"] *= scale
        v["frac"] *= scale
    step_prof_ms = sum(v[0] for v in prof.values())
    dom = max(table, key=lambda k: table[k]["ms_per_step"]) if table else None
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if dom and os.path.exists(tpath):
        traffic = json.load(open(tpath)).get(prob.name, {}).get(table[dom]["kernel"])
    model = byte_model(prob, args.n_cg, word)
    it_model_gbs = model["iteration"] * scale * (args.steps * ips) / (sum(lvl_ms[:1]) / 1e3) / 1e9

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        ts = oracle_sample(prob, args.cpu_iters)
        cpu = {"value": args.cpu_iters / sum(ts), "unit": "it/s", "cores": 1, "kind": "oracle",
               "sample": f"{args.cpu_iters} fixed-work iterations of {prob.name} at full size "
                         f"(single-threaded fp64 C oracle, {sum(ts):.1f} s)", **host_info()}
    if rank == 0:
        d = table[dom] if dom else None
        line = {
            "metric": "PARSDMM iterations/s", "value": value_job, "unit": "it/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_total / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32" if prob.dtype == "f32" else "f64",
            "data": "synthetic",
            "config": workload_config(prob, args, world),
            "pts_sets_per_s": value_job * prob.N * len(prob.sets) if levels == 1 else None,
            "iteration_model_gbs": it_model_gbs,
            "comm_ms_per_step": prof.get("comm", (0.0, 0))[0],
            "roofline": None if d is None else {
                "kernel": d["kernel"], "bound": "hbm", "achieved": d["achieved_gbs"],
                "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": d["frac"], "traffic": traffic,
                "peak_source": peaks["source"] + " copy bandwidth (burst)",
                "bytes_per_step": d["bytes_per_step"], "launches_per_step": d["launches"],
                "avg_launch_us": 1e3 * d["ms_per_step"] / d["launches"],
                "share_of_step": d["ms_per_step"] / step_prof_ms if step_prof_ms else None},
            "kernels": table,
            "kernel_ms_per_step": {k: v[0] for k, v in prof.items()},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_val, "unit": "it/s", "h2d_bytes_per_step": nbytes,
                    "d2h_bytes_per_step": nbytes},
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        if levels > 1:
            line["levels_ms_per_step"] = [v / args.steps for v in lvl_ms]
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def run_dry(args):
    """--dry-run: the rank plumbing only (gloo on the host, no GPU): every
    rank joins, max-over-ranks of a per-rank number, rank 0 prints n_gpus"""
    import torch.distributed as dist
    world, rank, _ = dist_init()
    if world > 1:
        dist.init_process_group("gloo")
    v = max_over_ranks(float(rank + 1), world)
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "max_over_ranks": v}), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def launch_ranks(args):
    """--gpus N without a launcher: re-exec this script under
    torch.distributed.run with N ranks (one per GPU) on 127.0.0.1"""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C4", choices=sorted(G.CONFIGS))
    ap.add_argument("--multilevel", action="store_true",
                    help="C5: the 3-level multilevel solve (Algorithm 3), iters-per-step per level")
    ap.add_argument("--null-work", action="store_true",
                    help="the config's sets on an 8x8(x8) grid: the latency floor of the launch structure")
    ap.add_argument("--iters-per-step", type=int, default=10)
    ap.add_argument("--n-cg", type=int, default=10)
    ap.add_argument("--impl", default="cuda", choices=["cuda", "reference"])
    ap.add_argument("--cpu-iters", type=int, default=3)
    ap.add_argument("--ref-iters", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dry-run", action="store_true", help="rank plumbing only (no GPU)")
    ap.add_argument("--virtual-ranks", type=int, default=1,
                    help="run the z-slab path with G slabs on the one GPU (diagnostic)")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "0"))
    if world == 0 and args.gpus > 1:
        return launch_ranks(args)
    if world and world != args.gpus:
        print(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
        return 2
    if args.dry_run:
        return run_dry(args)
    prob = G.CONFIGS[args.config]()
    if args.null_work:
        shape = (8, 8) if len(prob.shape) == 2 else (8, 8, 8)
        small = G.CONFIGS[args.config](shape=shape)
        small.name = prob.name + "-null"
        prob = small
    if args.multilevel and prob.n_levels == 1:
        print("bench.py: --multilevel needs a multilevel config (C5)", file=sys.stderr)
        return 2
    if args.impl == "reference":
        return run_reference(args, prob)
    return run_cuda(args, prob)


if __name__ == "__main__":
    sys.exit(main())
