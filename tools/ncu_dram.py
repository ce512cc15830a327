"""Per-kernel DRAM bytes / duration / throughput of an ncu --set full report
(run here, no GPU):  python tools/ncu_dram.py REP [TRAFFIC_JSON KERNEL_SUBSTR]
With the extra arguments also writes the bench.py traffic file for that kernel."""
import csv
import io
import json
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                      "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,"
                      "sm__throughput.avg.pct_of_peak_sustained_elapsed,"
                      "l1tex__throughput.avg.pct_of_peak_sustained_active,launch__registers_per_thread,"
                      "sm__warps_active.avg.pct_of_peak_sustained_active"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, units = rows[0], rows[1]
col = {n: i for i, n in enumerate(h)}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3}
res = []
for r in rows[2:]:
    def val(m):
        v = float(r[col[m]].replace(",", ""))
        return v * scale.get(units[col[m]], 1)
    rd, wr, t = val("dram__bytes_read.sum"), val("dram__bytes_write.sum"), val("gpu__time_duration.sum")
    res.append((r[col["Kernel Name"]], rd, wr, t))
    print(f"{r[col['Kernel Name']][:44]:44s} dram_read {rd / 1e6:9.3f} MB, write {wr / 1e6:9.3f} MB, time {t:9.2f} us, "
          f"sm {float(r[col['sm__throughput.avg.pct_of_peak_sustained_elapsed']]):5.1f}%, "
          f"l1 {float(r[col['l1tex__throughput.avg.pct_of_peak_sustained_active']]):5.1f}%, "
          f"regs {r[col['launch__registers_per_thread']]}, "
          f"occ {float(r[col['sm__warps_active.avg.pct_of_peak_sustained_active']]):5.1f}%")
if len(sys.argv) > 3:
    k = [x for x in res if sys.argv[3] in x[0]][0]
    json.dump({"kernel": k[0].split("(")[0] + " (ss_train_backward_records)",
               "source": f"{sys.argv[2].replace('_traffic.json', '_ncu_dram.txt')} (ncu --set full, one config-2 launch)",
               "dram_bytes_per_launch": int(k[1] + k[2]),
               "note": f"dram__bytes_read.sum + dram__bytes_write.sum = {k[1] / 1e6:.2f} MB + {k[2] / 1e6:.2f} MB"},
              open(sys.argv[2], "w"), indent=1)
