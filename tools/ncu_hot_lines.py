"""Dump SASS lines of one kernel with executed counts, for the address range
around the hottest lines.   python tools/ncu_hot_lines.py rep regex:k [min_count]"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
mn = float(sys.argv[3]) if len(sys.argv) > 3 else 1e7
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", kern],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
i0 = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[i0]
ie, src = h.index("Instructions Executed"), h.index("Source")
st = h.index("Warp Stall Sampling (All Samples)")
for k, r in enumerate(rows[i0 + 1:]):
    if len(r) <= ie or not r[0].startswith("0x"):
        break
    c = float(r[ie] or 0)
    if c >= mn:
        print(f"{k:5d} {c:12.4g} {r[st]:>6s}  {r[src].strip()[:110]}")
