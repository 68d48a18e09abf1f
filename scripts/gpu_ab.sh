# A/B of library variants (WS_LIB) in fused+graph mode, plus the persistent-kernel probe
for v in "" _mb3 _mb4; do WS_LIB=paper_2603_28381_b200/libwarpstar_b200$v.so timeout 300 python scripts/time_modes.py fused+graph persistent; done
WS_LIB=paper_2603_28381_b200/libwarpstar_b200_probe.so timeout 300 python scripts/persist_probe.py 2>&1 | tail -8
