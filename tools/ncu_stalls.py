"""Warp-stall reason breakdown of one kernel in an ncu --set full report."""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv", "--kernel-name", f"regex:{sys.argv[2]}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, v = rows[0], rows[2]
pre = "smsp__average_warps_issue_stalled_"
items = []
for k, x in zip(h, v):
    if k.startswith(pre) and k.endswith("_per_issue_active.ratio"):
        try:
            items.append((float(x), k[len(pre):-len("_per_issue_active.ratio")]))
        except ValueError:
            pass
tot = sum(a for a, _ in items) or 1
for a, k in sorted(items, reverse=True)[:12]:
    print(f"{k:28s} {a:7.2f} cycles/issue  {100 * a / tot:5.1f}%")
