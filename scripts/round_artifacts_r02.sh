# Round-2 evidence (run on a B200 from the repo root): GPU parity, smoke, the
# bench lines (ours + reference arm), the ncu launch list of the bench
# command, the per-pass DRAM traffic of one graph-replayed pass (app-range
# replay), the in-pass per-class times (WS_PROBE stamps), full ncu captures of
# the dominant kernels (single pass, 16-corner batch, fused position-gradient
# backward level), and the placement step's launch list.  Outputs under
# gpurun_out/; scripts/make_profiles.py r02 copies the summaries to profiles/.
R=${1:-r02}
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu_$R.txt
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > $O/pytest_gpu_$R.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu_$R.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_$R.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $O/bench_$R.json 2> $O/bench_$R.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref_$R.json 2> $O/bench_ref_$R.err; echo "ref rc=$?"
NB="--cpu-baseline 0 --placement 0 --corners 0 --dropin 0"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$R.csv python bench.py --steps 2 --warmup 1 $NB > /dev/null 2>&1; echo "launches rc=$?"
timeout 600 ncu --replay-mode app-range --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv --log-file $O/traffic_apprange_$R.csv python scripts/pass_range.py > $O/apprange.log 2>&1; echo "traffic rc=$?"
python scripts/traffic_range_json.py $R
WS_LIB=paper_2603_28381_b200/libwarpstar_b200_probe.so timeout 300 python scripts/inpass_profile.py $R $O/launches_$R.csv > $O/inpass_$R.log 2>&1; echo "inpass rc=$?"; tail -3 $O/inpass_$R.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fwd -s 30 -c 1 -o $O/prof_fwd_$R python bench.py --steps 1 --warmup 1 --graph 0 $NB > /dev/null 2>&1; echo "full fwd rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_bwd -s 30 -c 1 -o $O/prof_bwd_$R python bench.py --steps 1 --warmup 1 --graph 0 $NB > /dev/null 2>&1; echo "full bwd rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_rc_flat -s 1 -c 1 -o $O/prof_rc_$R python bench.py --steps 1 --warmup 1 --graph 0 $NB > /dev/null 2>&1; echo "full rc rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fwd -s 30 -c 1 -o $O/prof_fwd16_$R python scripts/time_corners.py 16 > /dev/null 2>&1; echo "full fwd16 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_bwd -s 30 -c 1 -o $O/prof_bwd16_$R python scripts/time_corners.py 16 > /dev/null 2>&1; echo "full bwd16 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/place_launches_$R.csv python scripts/place_step.py 2 > /dev/null 2>&1; echo "place launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_bwd -s 90 -c 1 -o $O/prof_bwdpg_$R python scripts/place_step.py 2 > /dev/null 2>&1; echo "full bwd-pg rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_wire -s 1 -c 1 -o $O/prof_wire_$R python scripts/place_step.py 2 > /dev/null 2>&1; echo "full wire rc=$?"
# summaries on the box (ncu is here), then drop the reports: gpurun_out/
# travels back only under 64 MiB
python scripts/make_profiles.py $R --out $O/profiles_$R
tar czf $O/ncu_reps_$R.tgz -C $O $(cd $O && ls prof_*_$R.ncu-rep | head -3) 2>/dev/null
rm -f $O/*.ncu-rep
du -sh $O; ls $O/ $O/profiles_$R
