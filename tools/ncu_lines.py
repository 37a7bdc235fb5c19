"""Warp-stall samples per CUDA source line of an ncu --set full report
(--import-source on, -lineinfo builds): the top lines of one kernel.

usage: python tools/ncu_lines.py report.ncu-rep [top=30]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
cur, h, agg = None, None, {}
for r in csv.reader(io.StringIO(raw)):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        h = r
        continue
    if h is None or r[0] == "Function Name" or len(r) < 8 or r[2] != "-":
        continue
    try:
        agg[(cur, int(r[0]))] = (int(r[4]), int(r[7]), r[1].strip()[:96])
    except ValueError:
        pass
tot = sum(v[0] for v in agg.values()) or 1
print(f"total stall samples {tot}")
for (f, ln), (smp, inst, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{smp:7d} {100 * smp / tot:5.1f}%  inst={inst:10d}  {f}:{ln}  {src}")
