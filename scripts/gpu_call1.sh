set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python scripts/time_modes.py fused+graph fused persistent streams+graph
WS_LIB=paper_2603_28381_b200/libwarpstar_b200_probe.so timeout 300 python scripts/fused_probe.py
