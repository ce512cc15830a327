"""Write the committed profile summaries of a gpu_prof2.sh run:
profiles/<tag>_launches.txt (per-kernel launch list summary),
profiles/<tag>_traffic.json (DRAM bytes per launch of the record backward,
the bench roofline kernel) and profiles/<tag>_ncu_full.txt (ncu --set full
key metrics of the main kernels)."""
import collections
import csv
import json
import subprocess
import sys

tag, src = sys.argv[1], sys.argv[2]   # e.g. r2, gpurun_out/..._r2b
rows = list(csv.reader(open(f"{src}.csv" if not src.endswith(".csv") else src)))
hdr_i = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr = rows[hdr_i]
ki, mi, vi, ui, idi = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
val, names = collections.defaultdict(dict), {}
scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "byte": 1.0,
         "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
for r in rows[hdr_i + 1:]:
    if len(r) > vi:
        val[r[idi]][r[mi]] = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        names[r[idi]] = r[ki].split("(")[0]
out = subprocess.run([sys.executable, "tools/launches2.py", src], capture_output=True, text=True).stdout
open(f"profiles/{tag}_launches.txt", "w").write(out)
REC = ("area_class_kernel", "area_scatter_kernel", "splat_bwd_kernel", "big_bwd_kernel", "big_finish_kernel",
       "pixel_ndc_kernel")
per = collections.defaultdict(lambda: [0, 0.0, 0.0])
for i, m in val.items():
    if any(k in names[i] for k in REC):
        base = [k for k in REC if k in names[i]][0]
        per[base][0] += 1
        per[base][1] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        per[base][2] += m.get("gpu__time_duration.sum", 0.0)
nview = per["splat_bwd_kernel"][0]
tot = sum(p[1] for p in per.values()) / max(nview, 1)
json.dump({"kernel": "record backward (ss_train_backward_records: area classes, splat_bwd, big rects)",
           "dram_bytes_per_launch": tot, "launches": nview,
           "per_kernel_bytes_per_view": {k: p[1] / max(nview, 1) for k, p in per.items()},
           "source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum ({src}), cold cache, serialised"},
          open(f"profiles/{tag}_traffic.json", "w"), indent=1)
print(out)
print("record backward DRAM bytes per launch:", tot)
