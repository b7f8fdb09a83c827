"""Per-source-line instruction and stall-sample shares of one kernel in an ncu
report captured with --import-source on (ncu --page source --print-source
cuda,sass: one aggregate row per CUDA line, then its SASS rows).

usage: python tools/ncu_lines.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = []
fname = None
hdr = None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0].isdigit():
        try:
            samp = float(r[6] or 0)      # "# Samples"
            inst = float(r[7] or 0)      # "Instructions Executed"
        except (ValueError, IndexError):
            continue
        if samp or inst:
            rows.append((fname, int(r[0]), samp, inst, r[1].strip()[:70]))
ts = sum(x[2] for x in rows) or 1
ti = sum(x[3] for x in rows) or 1
print(f"total warp-instructions {ti:.0f}, stall samples {ts:.0f}")
for f, ln, s, i, src in sorted(rows, key=lambda x: -x[2])[:top]:
    print(f"{f}:{ln:<5} samples {100 * s / ts:5.1f}%  inst {100 * i / ti:5.1f}%  {src}")
