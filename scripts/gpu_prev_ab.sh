# same-box A/B of the single-corner pass: the library before the batch changes (e12d647) vs the current one
cd $GRAFT_REPO_ROOT
for r in 1 2 3; do
  for v in _prev ""; do WS_LIB=paper_2603_28381_b200/libwarpstar_b200$v.so timeout 300 python scripts/time_corners.py 1 16 2>&1 | tail -1; done
done
for v in _prev ""; do WS_LIB=paper_2603_28381_b200/libwarpstar_b200$v.so timeout 300 python scripts/time_place.py 2>&1 | tail -1 | sed "s/^/$v /"; done
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu_r02.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_r02.log
