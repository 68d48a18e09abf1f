"""Top CUDA source lines by executed warp instructions in an ncu report
(with lane efficiency).  python scripts/ncu_instr.py rep.ncu-rep [n]"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
rows, cur, hdr = [], "?", None
for line in out.splitlines():
    if line.startswith('"File Path"'):
        cur = line.split('","')[1].rstrip('"').split("/")[-1]
        continue
    if line.startswith('"Function Name"'):
        continue
    r = next(csv.reader(io.StringIO(line)))
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 9 or r[2] != "-":     # CUDA-line aggregate rows only
        continue
    try:
        ie, te = float(r[7]), float(r[8])
    except ValueError:
        continue
    rows.append((ie, te, cur, r[0], r[1].strip()[:100]))
tot = sum(x[0] for x in rows) or 1
print(f"warp instructions {tot:.0f}, lane efficiency {sum(x[1] for x in rows) / tot / 32:.2f}")
for ie, te, f, ln, src in sorted(rows, reverse=True)[:n]:
    print(f"{ie:9.0f} {ie / tot:.3f} eff={te / max(ie, 1) / 32:.2f} {f}:{ln} {src}")
