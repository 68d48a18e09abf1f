"""Key metrics of an ncu report: python scripts/ncu_summary.py rep.ncu-rep"""
import csv
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct"]
STALL = "smsp__average_warps_issue_stalled_"
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, u = rows[0], rows[1]
for v in rows[2:]:
    print("kernel:", v[h.index("Kernel Name")][:80])
    for i, k in enumerate(h):
        if k in WANT:
            print(f"  {k:60s} {v[i]:>14s} {u[i]}")
    st = [(float(v[i]), k[len(STALL):]) for i, k in enumerate(h)
          if k.startswith(STALL) and k.endswith("_per_issue_active.ratio") and v[i] not in ("", "n/a")]
    st.sort(reverse=True)
    print("  top stalls (warps per issue):", ", ".join(f"{n.replace('_per_issue_active.ratio','')}={x:.2f}" for x, n in st[:6]))
