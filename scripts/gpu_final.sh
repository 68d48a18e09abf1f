# final checks on the final code: sanitizers (incl. split batches + RC fold), GPU suite, bench line
cd $GRAFT_REPO_ROOT
O=gpurun_out
{ echo '$ compute-sanitizer --tool memcheck python scripts/sanitize_run.py'; timeout 900 compute-sanitizer --tool memcheck python scripts/sanitize_run.py 2>&1 | grep -E "ERROR SUMMARY|ok$|Error" | tail -4
  echo '$ compute-sanitizer --tool racecheck python scripts/sanitize_run.py'; timeout 900 compute-sanitizer --tool racecheck python scripts/sanitize_run.py 2>&1 | grep -E "RACECHECK SUMMARY|ok$" | tail -4
  echo '$ compute-sanitizer --tool synccheck python scripts/sanitize_run.py'; timeout 900 compute-sanitizer --tool synccheck python scripts/sanitize_run.py 2>&1 | grep -E "ERROR SUMMARY|ok$" | tail -4; } > $O/sanitizer.txt 2>&1
cat $O/sanitizer.txt
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > $O/pytest_gpu_r02.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu_r02.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu_r02.txt
timeout 900 python bench.py > $O/bench_r02.json 2> $O/bench_r02.err; echo "bench rc=$?"; tail -c 400 $O/bench_r02.json
