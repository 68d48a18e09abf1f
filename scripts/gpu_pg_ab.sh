# A/B: fused position-gradient backward level kernel at 2 (default) vs 3 blocks/SM (WS_MINB_PG=3 build): C4 step and 16 candidates
cd $GRAFT_REPO_ROOT
for r in 1 2; do
  for v in "" _pg3; do
    WS_LIB=paper_2603_28381_b200/libwarpstar_b200$v.so timeout 300 python scripts/time_candidates.py 2>&1 | tail -1 | sed "s/^/lib=$v cand /"
    WS_LIB=paper_2603_28381_b200/libwarpstar_b200$v.so timeout 300 python scripts/time_place.py 2>&1 | tail -2 | sed "s/^/lib=$v place /"
  done
done
