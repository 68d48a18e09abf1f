"""Top CUDA source lines by warp-stall samples in an ncu report.

python scripts/ncu_lines.py report.ncu-rep [n]
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
cur_file = "?"
for line in out.splitlines():
    if line.startswith('"File Path"'):
        cur_file = line.split('","')[1].rstrip('"').split("/")[-1]
        continue
    if line.startswith('"Function Name"') or line.startswith('"Line No"'):
        continue
    r = next(csv.reader(io.StringIO(line)))
    if len(r) < 6 or r[2] != "-":
        continue          # keep CUDA-line aggregate rows only
    try:
        rows.append((float(r[4]), cur_file, int(r[0]), r[1].strip()))
    except ValueError:
        pass
tot = sum(x[0] for x in rows) or 1
print(f"{tot:.0f} samples")
for s, f, ln, src in sorted(rows, reverse=True)[:n]:
    print(f"{s:6.0f} {s / tot:5.3f} {f}:{ln:<5d} {src[:95]}")
