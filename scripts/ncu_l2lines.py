"""Top CUDA source lines by L2 global sectors (and excessive sectors) in an
ncu report.  python scripts/ncu_l2lines.py rep.ncu-rep [n]"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
rows, cur, hdr = [], "?", None
for line in out.splitlines():
    if line.startswith('"File Path"') or line.startswith('"File Name"'):
        cur = line.split('","')[1].rstrip('"').split("/")[-1]
        continue
    r = next(csv.reader(io.StringIO(line)))
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) or r[2] != "-":
        continue
    d = dict(zip(hdr[4:], r[4:]))
    def f(k):
        try:
            return float(d.get(k, 0) or 0)
        except ValueError:
            return 0.0
    rows.append((f("L2 Theoretical Sectors Global"), f("L2 Theoretical Sectors Global Excessive"),
                 f("L2 Theoretical Sectors Local"), f("L1 Wavefronts Shared"), f("L1 Wavefronts Shared Excessive"),
                 cur, r[0], r[1].strip()[:80]))
tg = sum(x[0] for x in rows); te = sum(x[1] for x in rows); tl = sum(x[2] for x in rows)
ts = sum(x[3] for x in rows); tse = sum(x[4] for x in rows)
print(f"L2 global sectors {tg:.0f} (excessive {te:.0f}), local {tl:.0f}; smem wavefronts {ts:.0f} (excessive {tse:.0f})")
for g, e, l, s, se, fn, ln, src in sorted(rows, reverse=True)[:n]:
    print(f"{g:10.0f} exc {e:9.0f} loc {l:8.0f}  {fn}:{ln} {src}")
print("-- by shared wavefronts")
for g, e, l, s, se, fn, ln, src in sorted(rows, key=lambda x: -x[3])[:12]:
    print(f"{s:10.0f} exc {se:9.0f}  {fn}:{ln} {src}")
