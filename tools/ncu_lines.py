"""Per-CUDA-source-line instructions and stall samples of one kernel in an
ncu report (run here, no GPU):  python tools/ncu_lines.py REP KERNEL_REGEX [TOP]"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name", f"regex:{kre}"], capture_output=True, text=True).stdout
fname, hdr, rows = "?", None, []
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] in ("", "Function Name"):
        continue
    try:
        ws = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
        ex = int(r[hdr.index("Instructions Executed")])
    except (ValueError, IndexError):
        continue
    rows.append((f"{fname}:{r[0]}", r[1].strip()[:90], ex, ws))
te = sum(x[2] for x in rows) or 1
tw = sum(x[3] for x in rows) or 1
print(f"warp instructions {te}, stall samples {tw}")
print("   instr%  stall%  line")
for loc, src, ex, ws in sorted(rows, key=lambda x: -x[3])[:top]:
    print(f"  {100 * ex / te:6.1f}  {100 * ws / tw:6.1f}  {loc:22s} {src}")
if len(sys.argv) > 4:   # group: file:lo-hi,...
    for spec in sys.argv[4].split(","):
        f, rng = spec.split(":")
        lo, hi = map(int, rng.split("-"))
        sel = [x for x in rows if x[0].split(":")[0] == f and lo <= int(x[0].split(":")[1]) <= hi]
        print(f"{spec:28s} instr {100 * sum(x[2] for x in sel) / te:5.1f}%  stall {100 * sum(x[3] for x in sel) / tw:5.1f}%")
