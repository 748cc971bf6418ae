"""Summarise an ncu report: key throughput metrics + top stall reasons (+ hot SASS regions)."""
import csv, subprocess, sys
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, u = rows[0], rows[1]
keys = ['Kernel Name', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active', 'l1tex__throughput.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'smsp__warps_eligible.avg.per_cycle_active', 'smsp__inst_executed.sum',
        'launch__occupancy_limit_shared_mem', 'launch__occupancy_limit_registers', 'launch__grid_size']
for r in rows[2:]:
    print('-' * 60)
    for k in keys:
        if k in h:
            i = h.index(k)
            print(f"  {k:62s} {r[i][:50]:>20s} {u[i]}")
    st = [i for i, x in enumerate(h) if x.startswith('smsp__pcsamp_warps_issue_stalled') and not x.endswith('not_issued')]
    vals = sorted([(h[i].replace('smsp__pcsamp_warps_issue_stalled_', ''), float(r[i].replace(',', '') or 0))
                   for i in st if r[i] not in ('', 'n/a')], key=lambda x: -x[1])[:6]
    tot = sum(v for _, v in vals) or 1
    print('  stalls:', ', '.join(f"{a} {100 * b / tot:.0f}%" for a, b in vals))
