# Round-end evidence: bench lines (ours + reference arm), ncu launch list of the
# bench command, per-pass DRAM traffic of every pass kernel, one full ncu
# capture of the dominant kernel.  Outputs under gpurun_out/ (copied to profiles/).
R=${1:-r01}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_$R.txt
timeout 900 python bench.py > gpurun_out/bench_$R.json 2> gpurun_out/bench_$R.err; echo "bench rc=$?"; cat gpurun_out/bench_$R.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$R.json 2> gpurun_out/bench_ref_$R.err; echo "ref rc=$?"; cat gpurun_out/bench_ref_$R.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$R.csv python bench.py --steps 2 --warmup 1 --cpu-baseline 0 > /dev/null 2>&1; echo "launches rc=$?"
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv -k "regex:^k_(free|rc_flat|rc_tree|fwd|bwd|fin|summary|pass)$" --kernel-name-base function -c 124 --log-file gpurun_out/traffic_$R.csv python bench.py --steps 1 --warmup 0 --graph 0 --cpu-baseline 0 > /dev/null 2>&1; echo "traffic rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fwd -s 30 -c 1 -o gpurun_out/prof_fwd_$R python bench.py --steps 1 --warmup 1 --graph 0 --cpu-baseline 0 > /dev/null 2>&1; echo "full fwd rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bwd -s 30 -c 1 -o gpurun_out/prof_bwd_$R python bench.py --steps 1 --warmup 1 --graph 0 --cpu-baseline 0 > /dev/null 2>&1; echo "full bwd rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rc_flat -s 1 -c 1 -o gpurun_out/prof_rc_$R python bench.py --steps 1 --warmup 1 --graph 0 --cpu-baseline 0 > /dev/null 2>&1; echo "full rc rc=$?"
ls -la gpurun_out/
