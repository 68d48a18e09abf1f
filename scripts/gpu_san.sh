cd $GRAFT_REPO_ROOT
timeout 300 python scripts/sanitize_run.py > gpurun_out/san_plain.log 2>&1; echo "plain rc=$?"; tail -15 gpurun_out/san_plain.log
timeout 900 compute-sanitizer --tool memcheck python scripts/sanitize_run.py > gpurun_out/san_mem.log 2>&1; echo "mem rc=$?"; tail -8 gpurun_out/san_mem.log
