"""Group the SASS of one kernel in an ncu report by execution count (loop
bodies show up as blocks of equal count): python tools/sass_counts.py REP KRE [N]"""
import collections
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass",
                      "--kernel-name", f"regex:{sys.argv[2]}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
for i, r in enumerate(rows):
    if 'Source' in r and 'Instructions Executed' in r:
        h, start = r, i + 1
        break
ei, wi = h.index('Instructions Executed'), h.index('Warp Stall Sampling (All Samples)')
c, st = collections.Counter(), collections.Counter()
for r in rows[start:]:
    try:
        n, w = int(r[ei]), int(r[wi])
    except (ValueError, IndexError):
        continue
    c[n] += 1
    st[n] += w
tot = sum(n * k for n, k in c.items())
tw = sum(st.values()) or 1
print(f"warp instructions {tot}")
for n, k in sorted(c.items(), key=lambda x: -x[0] * x[1])[:int(sys.argv[3]) if len(sys.argv) > 3 else 15]:
    print(f"count {n:9d} x {k:4d} instrs = {n * k / tot * 100:5.1f}% instr, {100 * st[n] / tw:5.1f}% stall")
