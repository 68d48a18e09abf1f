# split parts A/B (WS_SPLIT_PARTS 2 / 3 / 4) on 16-corner and 16-candidate batches; bitwise tests under 4 parts
cd $GRAFT_REPO_ROOT
for r in 1 2; do
  for v in 2 3 4; do
    WS_SPLIT_PARTS=$v timeout 300 python scripts/time_corners.py 16 2>&1 | tail -1 | sed "s/^/parts=$v /"
    WS_SPLIT_PARTS=$v timeout 300 python scripts/time_candidates.py 2>&1 | tail -1 | sed "s/^/parts=$v cand /"
  done
done
WS_SPLIT_PARTS=4 timeout 900 python -m pytest tests/test_gpu_batch.py tests/test_gpu_place.py -k "split or batch" -q -x -p no:cacheprovider 2>&1 | tail -2
