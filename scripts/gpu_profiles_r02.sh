# round-2 profile artefacts: launch list, in-pass classes, range-replay traffic, full captures
set -x
OUT=gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_(rc_flat|fwd|bwd|fin_summary)" -c 122 --csv --log-file $OUT/launches_r02.csv python bench.py --steps 1 --warmup 0 --graph 0 --cpu-baseline 0 --corners 0 --placement 0 --dropin 0 > $OUT/launches_bench.log 2>&1
WS_LIB=paper_2603_28381_b200/libwarpstar_b200_probe.so timeout 300 python scripts/inpass_profile.py r02 $OUT/launches_r02.csv > $OUT/inpass.log 2>&1
timeout 600 ncu --replay-mode range --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv --log-file $OUT/traffic_range_r02.csv python scripts/pass_range.py > $OUT/range.log 2>&1
timeout 600 ncu --replay-mode app-range --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv --log-file $OUT/traffic_apprange_r02.csv python scripts/pass_range.py > $OUT/apprange.log 2>&1
tail -n 5 $OUT/range.log $OUT/apprange.log $OUT/inpass.log
cat $OUT/traffic_range_r02.csv | tail -5
python scripts/traffic_range_json.py r02
cp $OUT/launches_r02.csv profiles/launches_r02.csv 2>/dev/null
python scripts/launches.py $OUT/launches_r02.csv > profiles/launches_r02.txt
