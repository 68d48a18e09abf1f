# full ncu captures of one fwd and one bwd level kernel inside a 16-corner
# batch (throughput regime) and a single-corner pass (latency regime)
set -x
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fwd -s 30 -c 1 -o gpurun_out/prof_fwd16 python scripts/time_corners.py 16 > gpurun_out/ncu_fwd16.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_bwd -s 30 -c 1 -o gpurun_out/prof_bwd16 python scripts/time_corners.py 16 > gpurun_out/ncu_bwd16.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fwd -s 30 -c 1 -o gpurun_out/prof_fwd1 python scripts/time_corners.py 1 > gpurun_out/ncu_fwd1.log 2>&1
ls -la gpurun_out
