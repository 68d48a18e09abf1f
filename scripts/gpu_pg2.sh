# batch-only 3-block PG kernel: candidates + C4 timing, placement/batch GPU tests
cd $GRAFT_REPO_ROOT
for r in 1 2; do
  timeout 300 python scripts/time_candidates.py 2>&1 | tail -1
  timeout 300 python scripts/time_place.py 2>&1 | tail -1
done
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu_r02.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_r02.log
