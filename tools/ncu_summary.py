"""Key metrics + top stall lines of an ncu --set full report (run here, no GPU)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
kfilter = sys.argv[2] if len(sys.argv) > 2 else None
KEEP = ('Duration', 'Compute (SM) Throughput', 'Memory Throughput', 'DRAM Throughput', 'L1/TEX Cache Throughput',
        'L2 Cache Throughput', 'Achieved Occupancy', 'Theoretical Occupancy', 'Registers Per Thread',
        'Executed Ipc Active', 'Issue Slots Busy', 'No Eligible', 'Eligible Warps Per Scheduler',
        'Warp Cycles Per Issued Instruction', 'Executed Instructions', 'L1/TEX Hit Rate', 'L2 Hit Rate',
        'Branch Efficiency', 'Local Memory Spilling Requests')
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
ki, mi, vi, ui = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value'), h.index('Metric Unit')
seen = set()
for r in rows[1:]:
    if kfilter and kfilter not in r[ki]:
        continue
    key = (r[ki], r[mi])
    if r[mi] in KEEP and key not in seen:
        seen.add(key)
        print(f"{r[ki][:40]:40s} | {r[mi]} = {r[vi]} {r[ui]}")
if len(sys.argv) > 3:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "--kernel-name", f"regex:{sys.argv[3]}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    h = rows[1]
    si, ei, wi = h.index('Source'), h.index('Instructions Executed'), h.index('Warp Stall Sampling (All Samples)')
    data = []
    for r in rows[2:]:
        try:
            data.append((r[si].strip(), int(r[ei]), int(r[wi])))
        except (ValueError, IndexError):
            pass
    tw = sum(d[2] for d in data) or 1
    te = sum(d[1] for d in data)
    print(f"instructions {te}, stall samples {tw}")
    for s, ex, ws in sorted(data, key=lambda d: -d[2])[:int(sys.argv[4]) if len(sys.argv) > 4 else 25]:
        print(f"{ex:10d} {100 * ws / tw:5.1f}%  {s}")
