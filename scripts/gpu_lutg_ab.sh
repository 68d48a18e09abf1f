# A/B: LUT pool staged in shared memory per block (default) vs read in place through L1 (WS_LUT_GLOBAL=1)
cd $GRAFT_REPO_ROOT
for r in 1 2 3; do
  for v in 0 1; do WS_LUT_GLOBAL=$v timeout 300 python scripts/time_corners.py 1 4 16 2>&1 | tail -1 | sed "s/^/lut_global=$v /"; done
done
