"""Executed warp-instructions per SASS opcode of one kernel in an ncu report
(needs --import-source / -lineinfo captures), plus the hottest windows.

    python tools/ncu_opmix.py report.ncu-rep regex:compose_tma [top]
"""
import collections
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", kern],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
i0 = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[i0]
ie, src = h.index("Instructions Executed"), h.index("Source")
ti = h.index("Thread Instructions Executed")
data = []
for r in rows[i0 + 1:]:
    if len(r) <= ie or not r[0].startswith("0x"):
        break  # next kernel instance
    data.append(r)
mix = collections.Counter()
tmix = collections.Counter()
for r in data:
    op = r[src].strip().split()
    if not op:
        continue
    o = op[0]
    if o.startswith("@"):
        o = op[1]
    mix[o.split(".")[0]] += float(r[ie] or 0)
    tmix[o.split(".")[0]] += float(r[ti] or 0)
tot = sum(mix.values())
print(f"{len(data)} SASS lines, {tot:.4g} warp-inst, {sum(tmix.values()) / max(tot, 1):.1f} threads/inst")
for o, c in mix.most_common(top):
    print(f"  {o:10s} {c:14.4g} {100 * c / tot:5.1f}%  lanes {tmix[o] / max(c, 1):4.1f}")
