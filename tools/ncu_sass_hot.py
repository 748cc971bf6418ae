"""Hot SASS regions of an ncu report (instructions executed per window)."""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None
args = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
if kern: args += ["-k", kern]
rows = list(csv.reader(subprocess.run(args, capture_output=True, text=True).stdout.splitlines()))
start = 2 if rows[0][0] == 'Kernel Name' else 1
h = rows[start - 1]
ie, src = h.index('Instructions Executed'), h.index('Source')
data = [r for r in rows[start:] if len(r) > ie]
cnt = [float(r[ie] or 0) for r in data]
tot = sum(cnt)
win = int(sys.argv[3]) if len(sys.argv) > 3 else 50
regs = sorted(((sum(cnt[i:i + win]), i) for i in range(0, len(cnt), win)), reverse=True)[:int(sys.argv[4]) if len(sys.argv) > 4 else 8]
print(f"total {tot:.3g} warp-inst over {len(data)} SASS lines")
for s, i in regs:
    print(f"--- {i}-{i + win}: {100 * s / tot:.1f}%")
    if len(sys.argv) > 5:
        for j in range(i, min(i + win, len(data))):
            print(f"   {cnt[j]:10.0f} {data[j][src][:90]}")
