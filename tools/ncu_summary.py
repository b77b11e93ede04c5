"""Summarise an .ncu-rep (details page) per kernel launch."""
import csv
import subprocess
import sys

WANT = ['Duration', 'DRAM Throughput', 'Compute (SM) Throughput', 'Achieved Occupancy',
        'Registers Per Thread', 'Executed Ipc Active', 'L1/TEX Hit Rate', 'L2 Hit Rate',
        'Warp Cycles Per Issued Instruction', 'Executed Instructions', 'Theoretical Occupancy',
        'Memory Throughput']
rep = sys.argv[1]
out = subprocess.run(['ncu', '-i', rep, '--page', 'details', '--csv'], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[0]
ki, mi, vi, ui, idi = (h.index(x) for x in ('Kernel Name', 'Metric Name', 'Metric Value', 'Metric Unit', 'ID'))
rows = {}
for row in r[1:]:
    if row[mi] in WANT:
        d = rows.setdefault(row[idi], {'kernel': row[ki].split('(')[0]})
        d[row[mi] + (' (' + row[ui] + ')' if row[mi] == 'Memory Throughput' else '')] = row[vi]
for i, d in sorted(rows.items(), key=lambda t: int(t[0])):
    print(i, d.pop('kernel'))
    print('   ' + '; '.join(f'{k}={v}' for k, v in d.items()))
raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
hh = rr[0]
for row in rr[2:]:
    name = row[hh.index('Kernel Name')].split('(')[0]
    stalls = []
    for j, n in enumerate(hh):
        if n.startswith('smsp__average_warps_issue_stalled') and n.endswith('per_issue_active.ratio'):
            try:
                v = float(row[j].replace(',', ''))
            except ValueError:
                continue
            if v > 0.5:
                stalls.append((v, n.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')))
    db = [row[hh.index(n)] for n in ('dram__bytes_read.sum', 'dram__bytes_write.sum')]
    print(row[hh.index('ID')], name, 'dram R/W', db, 'stalls', sorted(stalls, reverse=True)[:4])
