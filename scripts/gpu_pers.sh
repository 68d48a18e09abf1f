timeout 120 python scripts/time_modes.py persistent || echo "persistent TIMEOUT/FAIL"
timeout 400 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
timeout 120 python scripts/time_modes.py fused+graph persistent
WS_LIB=paper_2603_28381_b200/libwarpstar_b200_probe.so timeout 120 python scripts/persist_probe.py 2>&1 | tail -7
