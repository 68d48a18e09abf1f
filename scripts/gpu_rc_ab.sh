# A/B: star-net root loads folded in the RC member blocks (default) vs separate net blocks (WS_RC_ROOTS=net); then the GPU suite
cd $GRAFT_REPO_ROOT
for r in 1 2 3; do
  for v in net fold; do WS_RC_ROOTS=$v timeout 300 python scripts/time_corners.py 1 16 2>&1 | tail -1 | sed "s/^/roots=$v /"; done
done
for v in net fold; do WS_RC_ROOTS=$v timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_rc_flat -c 3 python scripts/time_corners.py 1 2>&1 | grep -E "duration|bytes" | tail -3 | sed "s/^/roots=$v /"; done
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
