"""Per-kernel averages of an ncu launch-list CSV with several metrics
(gpu__time_duration.sum, dram__bytes_read.sum, dram__bytes_write.sum)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr_i = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr = rows[hdr_i]
ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
idi = hdr.index("ID")
val = collections.defaultdict(dict)
names = {}
for r in rows[hdr_i + 1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(",", ""))
    u = r[ui]
    v *= {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
          "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(u, 1.0)
    val[r[idi]][r[mi]] = v
    names[r[idi]] = r[ki].split("(")[0][:60]
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for i, m in val.items():
    a = agg[names[i]]
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0.0)
    a[2] += m.get("dram__bytes_read.sum", 0.0)
    a[3] += m.get("dram__bytes_write.sum", 0.0)
T = sum(a[1] for a in agg.values())
print(f"{'ms total':>9} {'share':>6} {'n':>4} {'ms/launch':>9} {'MB rd/l':>8} {'MB wr/l':>8} {'GB/s':>7}  kernel")
for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
    n, t, rd, wr = a
    print(f"{t:9.3f} {100 * t / T:5.1f}% {n:4d} {t / n:9.4f} {rd / n / 1e6:8.1f} {wr / n / 1e6:8.1f} "
          f"{(rd + wr) / (t / 1e3) / 1e9 if t else 0:7.0f}  {k}")
print(f"total {T:.3f} ms (cold-cache, serialised launches)")
