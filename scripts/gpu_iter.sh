# iteration: gpu parity, run-mode timing, persistent probe, fused launch list
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python scripts/check_modes.py
WS_LIB=paper_2603_28381_b200/libwarpstar_b200_probe.so timeout 300 python scripts/persist_probe.py 2>&1 | tail -7
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:k_(free|rc|fwd|bwd|fin|summary|pass)" -c 130 --csv --log-file gpurun_out/launches_fused.csv python bench.py --steps 1 --warmup 0 --graph 0 --cpu-baseline 0 > /dev/null 2>&1; python scripts/launches.py gpurun_out/launches_fused.csv | head -12
