"""Copy a round's GPU evidence from gpurun_out/ into profiles/ (tracked):
bench lines, launch-list summary, and text summaries of the full ncu captures.

python scripts/make_profiles.py r01
"""
import os
import shutil
import subprocess
import sys

R = sys.argv[1]
HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(HERE, "gpurun_out")
# --out DIR: write the summaries there (on a GPU box: under gpurun_out/, the
# only directory that travels back; the .ncu-rep files are too big to)
P = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else os.path.join(HERE, "profiles")
os.makedirs(P, exist_ok=True)
for f in (f"bench_{R}.json", f"bench_ref_{R}.json", f"gpu_{R}.txt", f"inpass_{R}.json"):
    if os.path.exists(os.path.join(G, f)):
        shutil.copy(os.path.join(G, f), os.path.join(P, f))
py = sys.executable
lc = os.path.join(G, f"launches_{R}.csv")
if os.path.exists(lc):
    out = subprocess.run([py, os.path.join(HERE, "scripts", "launches.py"), lc], capture_output=True, text=True).stdout
    with open(os.path.join(P, f"launches_{R}.txt"), "w") as fh:
        fh.write("# ncu --metrics gpu__time_duration.sum --clock-control none, command:\n"
                 "#   python bench.py --steps 2 --warmup 1 --cpu-baseline 0  (includes the one-time device build)\n"
                 "# per-launch times are cold-cache and serialised: compare shares, not absolutes\n")
        fh.write(out)
    shutil.copy(lc, os.path.join(P, f"launches_{R}.csv"))
for k in ("fwd", "bwd", "rc", "pglevel", "pgmem", "wire", "fwd16", "bwd16", "bwdpg"):
    rep = os.path.join(G, f"prof_{k}_{R}.ncu-rep")
    if not os.path.exists(rep):
        continue
    s = subprocess.run([py, os.path.join(HERE, "scripts", "ncu_summary.py"), rep], capture_output=True, text=True).stdout
    d = subprocess.run(["ncu", "-i", rep, "--page", "details"], capture_output=True, text=True).stdout
    with open(os.path.join(P, f"ncu_{k}_{R}.txt"), "w") as fh:
        fh.write(f"# ncu --set full --clock-control none --import-source on (one launch), {os.path.basename(rep)}\n")
        fh.write(s)
        for tool in ("ncu_stalls.py", "ncu_instr.py"):
            fh.write(f"\n# scripts/{tool} (top source lines)\n")
            fh.write(subprocess.run([py, os.path.join(HERE, "scripts", tool), rep, "20"], capture_output=True,
                                    text=True).stdout)
        fh.write("\n# --page details\n")
        fh.write(d)
# placement step: the last step's launches (wire + pass + position gradients)
pc = os.path.join(G, f"place_launches_{R}.csv")
if os.path.exists(pc):
    import collections
    import csv
    rows = list(csv.reader(open(pc)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, ii, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "ID", "Metric Name", "Metric Value", "Metric Unit"))
    per = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        d = per.setdefault(int(r[ii]), {"name": r[ki].split("(")[0].replace("(anonymous namespace)::", "")})
        v = float(r[vi].replace(",", ""))
        u = r[ui]
        if r[mi] == "gpu__time_duration.sum":
            v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(u, 1.0)
        elif u in ("Kbyte", "Mbyte", "Gbyte", "byte", "KB", "MB", "GB", "B"):
            v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}[u]
        d[r[mi]] = v
    ids = list(per)
    wire = [i for i in ids if per[i]["name"].endswith("k_wire")]
    last = [per[i] for i in ids if i >= wire[-1]] if wire else []
    agg = collections.OrderedDict()
    for d in last:
        a = agg.setdefault(d["name"], [0, 0.0, 0.0])
        a[0] += 1
        a[1] += d.get("gpu__time_duration.sum", 0.0)
        a[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    tot = sum(a[1] for a in agg.values()) or 1.0
    with open(os.path.join(P, f"place_launches_{R}.txt"), "w") as fh:
        fh.write("# ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum\n"
                 "#   --clock-control none, python scripts/place_step.py 2: the second C3 placement step\n"
                 "# (k_wire -> pass -> position gradients); cold-cache serialised: read shares\n")
        fh.write(f"{len(last)} launches, {tot:.1f} us total\n")
        for k, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
            fh.write(f"{k[:44]:44s} n={n:4d} total={t:9.1f}us avg={t / n:8.2f}us share={t / tot:.3f} "
                     f"dram={b / 1e6:9.2f}MB\n")
print(sorted(os.listdir(P)))
