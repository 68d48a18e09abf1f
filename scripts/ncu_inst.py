"""Top CUDA source lines by executed warp instructions in an ncu report.

python scripts/ncu_inst.py report.ncu-rep [n]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = []
cur = "?"
col = None
for line in out.splitlines():
    r = next(csv.reader(io.StringIO(line)))
    if r and r[0] == "File Path" or (r and r[0] == "File Name"):
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        col = r.index("Instructions Executed")
        continue
    if col is None or len(r) <= col or r[2] != "-":
        continue
    try:
        rows.append((float(r[col]), cur, int(r[0]), r[1].strip()))
    except ValueError:
        pass
tot = sum(x[0] for x in rows) or 1
print(f"{tot:.0f} warp instructions")
for s, f, ln, src in sorted(rows, reverse=True)[:n]:
    print(f"{s:10.0f} {s / tot:5.3f} {f}:{ln:<5d} {src[:90]}")
