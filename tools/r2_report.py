"""Assemble profiles/r02_final_c4.md from tools/gpu_final_r2.sh's outputs in
gpurun_out/ (bench lines, the ncu launch list with per-launch DRAM bytes, the
ncu --set full capture) and refresh profiles/ncu_traffic.json."""
import collections
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")
title = sys.argv[1] if len(sys.argv) > 1 else "Round 2 -- final measurements (one B200)"


def sh(cmd):
    return subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT).stdout


out = [f"# {title}", "",
       "Commands: `tools/gpu_final_r2.sh` (bench lines of every config, the C4 launch list with",
       "per-launch DRAM bytes, ncu --set full of the hot kernels, the Fig. 1 experiment, smoke());",
       "this file by `tools/r2_report.py`.", "",
       "## bench lines (device-timed, L2 flushed between steps; `kernels` = algorithmic GB/s per kernel kind)", "",
       "```"]
cfgs = ["C4", "C5", "C5_ml", "C3", "C2", "C1", "C1_null"]
for c in cfgs:
    src = os.path.join(G, f"r2_bench_{c}.json")
    if os.path.exists(src):
        shutil.copy(src, os.path.join(P, f"r02_final_bench_{c}.json"))
out.append(sh([sys.executable, "tools/bench_brief.py"] + [f"profiles/r02_final_bench_{c}.json" for c in cfgs
                                                          if os.path.exists(os.path.join(P, f"r02_final_bench_{c}.json"))]).rstrip())
out += ["```", ""]
ref = os.path.join(G, "r2_bench_reference.json")
if os.path.exists(ref):
    shutil.copy(ref, os.path.join(P, "r02_final_bench_reference.json"))
    for line in open(ref):
        if line.startswith("{"):
            d = json.loads(line)
            out += [f"Reference arm (the CPU oracle, fp64, {d['cpu_baseline']['cores']} thread, on the box's host): "
                    f"{d['value']:.4f} it/s on C4 (`r02_final_bench_reference.json`).", ""]
smoke = os.path.join(G, "r2_smoke.log")
if os.path.exists(smoke):
    shutil.copy(smoke, os.path.join(P, "r02_final_smoke.log"))

# launch list
lst = os.path.join(G, "r2_launches_c4.csv")
traffic = {}
if os.path.exists(lst):
    txt = [l for l in open(lst) if not l.startswith("==")]
    rows = list(csv.DictReader(io.StringIO("".join(txt))))
    per = collections.OrderedDict()
    for r in rows:
        mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3,
                "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3}.get(r["Metric Unit"], 1)
        per.setdefault(r["ID"], {"name": r["Kernel Name"].split("(")[0].replace("void ", "")})[r["Metric Name"]] = \
            float(r["Metric Value"].replace(",", "")) * mult
    agg = collections.OrderedDict()
    for d in per.values():
        a = agg.setdefault(d["name"], [0, 0.0, 0.0])
        a[0] += 1
        a[1] += d.get("gpu__time_duration.sum", 0.0)
        a[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    tot = sum(a[1] for a in agg.values())
    out += ["## C4 launch list (ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum",
            "--clock-control none; cold-cache, serialised; 2 steps = 20 iterations + warm-up)", "",
            "| kernel | launches | total us | avg us | share | DRAM MB / launch |", "|---|---|---|---|---|---|"]
    for k, (n, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"| `{k}` | {n} | {t:.1f} | {t / n:.2f} | {100 * t / tot:.1f}% | {b / n / 1e6:.1f} |")
        base = k.split("<")[0].replace("sip::", "")
        tb = traffic.setdefault(base, [0, 0.0])
        tb[0] += n
        tb[1] += b
    out.append(f"| total | {sum(a[0] for a in agg.values())} | {tot:.1f} | | 100% | |")
    out.append("")
    tj = {"C4": {k: v[1] / v[0] for k, v in traffic.items()}}
    tj["C4"]["k_selB+k_selC"] = (traffic.get("k_selB", [1, 0])[1] / max(1, traffic.get("k_selB", [1, 0])[0]) +
                                 3 * traffic.get("k_selC", [1, 0])[1] / max(1, traffic.get("k_selC", [1, 0])[0]))
    tj["C4"]["_about"] = ("dram__bytes_read.sum + dram__bytes_write.sum per launch (k_selB+k_selC: one k_selB "
                          "and three k_selC rounds), ncu launch list of profiles/r02_final_c4.md")
    json.dump(tj, open(os.path.join(P, "ncu_traffic.json"), "w"), indent=1)

sums = sorted(f for f in os.listdir(G) if f.startswith("r2_full") and f.endswith(".summary.txt"))
reps = sorted(f for f in os.listdir(G) if f.startswith("r2_full") and f.endswith(".ncu-rep"))
if sums:   # made on the GPU box by tools/gpu_final_r2.sh (the reports themselves may not travel back)
    out += ["## ncu --set full --import-source on, hot kernels of a C4 step (`tools/ncu_summary.py`)", "", "```"]
    for f in sums:
        out.append(open(os.path.join(G, f)).read().rstrip())
    out += ["```", ""]
elif reps:
    out += ["## ncu --set full --import-source on, hot kernels of a C4 step (`tools/ncu_summary.py`)", "", "```"]
    for f in reps:
        out.append(sh([sys.executable, "tools/ncu_summary.py", os.path.join(G, f)]).rstrip())
    out += ["```", ""]
fig = os.path.join(G, "r2_fig1_dykstra.json")
if os.path.exists(fig):
    shutil.copy(fig, os.path.join(P, "r02_fig1_dykstra.json"))
open(os.path.join(P, "r02_final_c4.md"), "w").write("\n".join(out) + "\n")
print("\n".join(out))
