# One full ncu capture per hot kernel (k_fwd, k_bwd, k_rc) on C3.
set -x
B="python bench.py --steps 1 --warmup 1 --graph 0 --cpu-baseline 0 --mode fused"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fwd -s 30 -c 1 -o gpurun_out/prof_fwd $B > gpurun_out/ncu_fwd.log 2>&1; echo "fwd rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bwd -s 30 -c 1 -o gpurun_out/prof_bwd $B > gpurun_out/ncu_bwd.log 2>&1; echo "bwd rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rc -s 0 -c 1 -o gpurun_out/prof_rc $B > gpurun_out/ncu_rc.log 2>&1; echo "rc rc=$?"
ls -la gpurun_out/
