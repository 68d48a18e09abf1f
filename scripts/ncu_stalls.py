"""Top CUDA source lines by warp-stall samples in an ncu report, with the
main stall reasons.  python scripts/ncu_stalls.py rep.ncu-rep [n]"""
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
    try:
        s = float(d["Warp Stall Sampling (All Samples)"])
    except ValueError:
        continue
    reasons = []
    for k in hdr:
        if k.startswith("stall_") and "Not Issued" not in k:
            try:
                v = float(d.get(k, 0) or 0)
            except ValueError:
                v = 0
            if v:
                reasons.append((v, k[6:]))
    reasons.sort(reverse=True)
    rows.append((s, cur, r[0], r[1].strip()[:90], reasons[:3]))
tot = sum(x[0] for x in rows) or 1
rows.sort(reverse=True)
print(f"stall samples {tot:.0f}")
for s, f, ln, src, rs in rows[:n]:
    print(f"{s / tot:6.3f} {f}:{ln} {src}\n        " + ", ".join(f"{k}={v / s:.2f}" for v, k in rs))
