"""one-screen summary of bench.py JSON lines"""
import json
import sys
for path in sys.argv[1:]:
    for line in open(path):
        if not line.startswith("{"):
            continue
        d = json.loads(line)
        rl = d.get("roofline") or {}
        print(f"== {path}: {d['value']:.1f} it/s  {d['ms_per_step']:.3f} ms/step  e2e {d['e2e']['value']:.1f}  "
              f"roofline {rl.get('kernel')} {rl.get('frac') or 0:.3f}  clocks {d.get('clocks', {}).get('sm_mhz')}")
        for k, v in d.get("kernels", {}).items():
            print(f"   {k:7s} {v['ms_per_step']:8.3f} ms {v['achieved_gbs']:7.0f} GB/s {v['frac']:.3f}")
        if "levels_ms_per_step" in d:
            print("   levels", [round(x, 2) for x in d["levels_ms_per_step"]])
