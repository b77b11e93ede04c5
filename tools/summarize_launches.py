"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) per kernel."""
import collections
import csv
import sys

path = sys.argv[1]
rows = list(csv.reader(open(path)))
hdr = None
agg = collections.OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = d["Kernel Name"].split("(")[0].replace("void ", "")
    v = float(d["Metric Value"].replace(",", ""))
    unit = d.get("Metric Unit", "ns")
    v = v / 1e3 if unit == "ns" else (v if unit == "us" else v * 1e3)   # -> us
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += v
tot = sum(a[1] for a in agg.values())
print(f"| kernel | launches | total us | avg us | share |")
print("|---|---|---|---|---|")
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"| `{k}` | {n} | {t:.1f} | {t / n:.2f} | {100 * t / tot:.1f}% |")
print(f"| total | {sum(a[0] for a in agg.values())} | {tot:.1f} | | 100% |")
