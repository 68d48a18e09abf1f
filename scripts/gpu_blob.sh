set -x
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
timeout 300 python scripts/time_modes.py fused+graph persistent
WS_LIB=paper_2603_28381_b200/libwarpstar_b200_probe.so timeout 300 python scripts/fused_probe.py 2>&1 | head -9
