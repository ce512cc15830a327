"""Summarise an ncu launch-list CSV (gpu__time_duration.sum per launch)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr_i = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr = rows[hdr_i]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
tot, cnt = collections.defaultdict(float), collections.Counter()
for r in rows[hdr_i + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0][:70]
    v = float(r[vi].replace(",", ""))
    v *= {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}.get(r[ui], 1.0)
    tot[name] += v
    cnt[name] += 1
T = sum(tot.values())
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{v:9.3f} ms {100 * v / T:5.1f}%  n={cnt[k]:4d}  {k}")
print(f"total {T:.3f} ms")
