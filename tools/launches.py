"""Print an ncu --metrics gpu__time_duration.sum --csv launch list (in order)."""
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if r]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for i, r in enumerate(rows):
    if 'Kernel Name' in r:
        h = r; start = i + 1; break
ki, vi, idi = h.index('Kernel Name'), h.index('Metric Value'), h.index('ID')
for r in rows[start:start + n]:
    if len(r) <= vi: continue
    name = r[ki].split('(')[0].replace('(anonymous namespace)::', '').replace('unnamed>::', '')
    print(f"{int(r[idi]):4d} {float(r[vi].replace(',', '')) / 1e6:9.3f} ms  {name}")
