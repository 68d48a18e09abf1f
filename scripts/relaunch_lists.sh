R=r01
NB="--cpu-baseline 0 --placement 0 --corners 0"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$R.csv python bench.py --steps 2 --warmup 1 $NB > /dev/null 2>&1; echo "launches rc=$?"
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv -k "regex:^k_(free|rc_flat|rc_tree|fwd|bwd|fin|summary|fin_summary|pass)$" --kernel-name-base function -c 122 --log-file gpurun_out/traffic_$R.csv python bench.py --steps 1 --warmup 0 --graph 0 $NB > /dev/null 2>&1; echo "traffic rc=$?"
