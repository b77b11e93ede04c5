"""Brief per-launch summary of an ncu report (ncu -i ... --page details --csv)."""
import csv
import subprocess
import sys

WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "Registers Per Thread", "Achieved Occupancy",
        "Executed Instructions", "Warp Cycles Per Issued Instruction", "L2 Hit Rate", "L1/TEX Hit Rate",
        "Compute (SM) Throughput", "Grid Size", "Dynamic Shared Memory Per Block", "Static Shared Memory Per Block"]


def main(path, filt=""):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    ki, mi, vi, ii, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID"), h.index("Metric Unit")
    cur = None
    for r in rows[1:]:
        if filt and filt not in r[ki]:
            continue
        if r[mi] in WANT:
            key = (r[ii], r[ki][:48])
            if key != cur:
                print("\n", key)
                cur = key
            print(f"    {r[mi]} = {r[vi]} {r[ui]}")


if __name__ == "__main__":
    main(*sys.argv[1:])
