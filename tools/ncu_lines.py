"""Per-source-line warp-stall samples of one kernel in an ncu report.

    python tools/ncu_lines.py report.ncu-rep [top]
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg, src = collections.Counter(), {}
f = line = None
for r in csv.reader(io.StringIO(out)):
    if r and r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if not r or r[0] in ("Function Name", "Line No"):
        continue
    if r[0] != "":
        line = r[0]
        src[(f, line)] = r[1]
        continue
    try:
        agg[(f, line)] += float(r[4])
    except (ValueError, IndexError):
        pass
tot = sum(agg.values()) or 1.0
print(f"total samples {tot:.0f}")
for k, v in agg.most_common(top):
    print(f"{v:7.0f} {100 * v / tot:5.1f}% {k[0]}:{k[1]} {src.get(k, '')[:96]}")
