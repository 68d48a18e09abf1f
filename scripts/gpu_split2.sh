# split (default, >= 8) vs lockstep (WS_SPLIT=0): corner and candidate batches; then the GPU suite
cd $GRAFT_REPO_ROOT
for r in 1 2; do
  for v in 0 8; do
    WS_SPLIT=$v timeout 300 python scripts/time_corners.py 1 8 16 2>&1 | tail -1 | sed "s/^/split=$v /"
    WS_SPLIT=$v timeout 300 python scripts/time_candidates.py 2>&1 | tail -1 | sed "s/^/split=$v cand /"
  done
done
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
