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
P = os.path.join(HERE, "profiles")
os.makedirs(P, exist_ok=True)
for f in (f"bench_{R}.json", f"bench_ref_{R}.json", f"gpu_{R}.txt"):
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
for k in ("fwd", "bwd", "rc"):
    rep = os.path.join(G, f"prof_{k}_{R}.ncu-rep")
    if not os.path.exists(rep):
        continue
    s = subprocess.run([py, os.path.join(HERE, "scripts", "ncu_summary.py"), rep], capture_output=True, text=True).stdout
    d = subprocess.run(["ncu", "-i", rep, "--page", "details"], capture_output=True, text=True).stdout
    with open(os.path.join(P, f"ncu_{k}_{R}.txt"), "w") as fh:
        fh.write(f"# ncu --set full --clock-control none --import-source on (one launch), {os.path.basename(rep)}\n")
        fh.write(s)
        fh.write("\n# --page details\n")
        fh.write(d)
print(sorted(os.listdir(P)))
