"""Per-source-line totals (instructions executed, stall samples) of an ncu
report captured with --import-source on and -lineinfo.  Inlined helpers are
attributed to their own lines."""
import csv, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows, path, hdr = [], "?", None
for r in csv.reader(out):
    if not r:
        continue
    if r[0] == "File Path":
        path = r[1].split("/")[-1]
    elif r[0] == "Line No":
        hdr = r
    elif hdr and len(r) > 8 and r[2] == "-":
        ie = hdr.index("Instructions Executed")
        sm = hdr.index("Warp Stall Sampling (All Samples)")
        try:
            rows.append((float(r[ie] or 0), float(r[sm] or 0), path, r[0], r[1].strip()[:80]))
        except ValueError:
            pass
ti = sum(x[0] for x in rows) or 1
ts = sum(x[1] for x in rows) or 1
print(f"total inst {ti:.3g}, samples {ts:.3g}")
for i, s, p, ln, src in sorted(rows, reverse=True)[:top]:
    print(f"{100 * i / ti:5.1f}% inst {100 * s / ts:5.1f}% stall  {p}:{ln}  {src}")
