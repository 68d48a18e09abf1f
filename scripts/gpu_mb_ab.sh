# A/B of the corner-batch level kernels' min blocks per SM (WS_MINB_BATCH 4 default vs 3 / 2 builds)
cd $GRAFT_REPO_ROOT
for r in 1 2; do
  for v in "" _mb3 _mb2; do WS_LIB=paper_2603_28381_b200/libwarpstar_b200$v.so timeout 300 python scripts/time_corners.py 4 16 2>&1 | tail -1; done
done
