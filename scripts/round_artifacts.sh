# Round-end evidence: bench lines (ours + reference arm), ncu launch list of the
# bench command, per-pass DRAM traffic of every pass kernel, full ncu captures
# of the dominant kernels, and the placement step's launch list + captures.
# Outputs under gpurun_out/ (copied to profiles/ by scripts/make_profiles.py).
R=${1:-r01}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_$R.txt
timeout 600 python bench.py > gpurun_out/bench_$R.json 2> gpurun_out/bench_$R.err; echo "bench rc=$?"; cat gpurun_out/bench_$R.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$R.json 2> gpurun_out/bench_ref_$R.err; echo "ref rc=$?"; cat gpurun_out/bench_ref_$R.json
NB="--cpu-baseline 0 --placement 0 --corners 0"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$R.csv python bench.py --steps 2 --warmup 1 $NB > /dev/null 2>&1; echo "launches rc=$?"
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv -k "regex:^k_(free|rc_flat|rc_tree|fwd|bwd|fin|summary|fin_summary|pass)$" --kernel-name-base function -c 122 --log-file gpurun_out/traffic_$R.csv python bench.py --steps 1 --warmup 0 --graph 0 $NB > /dev/null 2>&1; echo "traffic rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fwd -s 30 -c 1 -o gpurun_out/prof_fwd_$R python bench.py --steps 1 --warmup 1 --graph 0 $NB > /dev/null 2>&1; echo "full fwd rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_bwd -s 30 -c 1 -o gpurun_out/prof_bwd_$R python bench.py --steps 1 --warmup 1 --graph 0 $NB > /dev/null 2>&1; echo "full bwd rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_rc_flat -s 1 -c 1 -o gpurun_out/prof_rc_$R python bench.py --steps 1 --warmup 1 --graph 0 $NB > /dev/null 2>&1; echo "full rc rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/place_launches_$R.csv python scripts/place_step.py 2 > /dev/null 2>&1; echo "place launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pg_level -s 90 -c 1 -o gpurun_out/prof_pglevel_$R python scripts/place_step.py 2 > /dev/null 2>&1; echo "full pg_level rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pg_mem -s 90 -c 1 -o gpurun_out/prof_pgmem_$R python scripts/place_step.py 2 > /dev/null 2>&1; echo "full pg_mem rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_wire -s 1 -c 1 -o gpurun_out/prof_wire_$R python scripts/place_step.py 2 > /dev/null 2>&1; echo "full wire rc=$?"
ls -la gpurun_out/
