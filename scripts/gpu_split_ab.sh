# A/B: fused corner batches as two half batches on two streams (WS_SPLIT=n) vs one lockstep batch; batch tests under the split
cd $GRAFT_REPO_ROOT
for r in 1 2 3; do
  for v in 0 8 4; do WS_SPLIT=$v timeout 300 python scripts/time_corners.py 4 8 16 2>&1 | tail -1 | sed "s/^/split=$v /"; done
done
WS_SPLIT=4 timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_gpu_full.py -k batch -q -x -p no:cacheprovider 2>&1 | tail -2
