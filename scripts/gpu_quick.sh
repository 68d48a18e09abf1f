# quick GPU iteration: parity subset + bench modes + phase probe
set -x
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
for m in persistent fused streams; do timeout 300 python bench.py --steps 20 --warmup 5 --cpu-baseline 0 --mode $m 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$m', d['value'], 'e2e', d['e2e']['value'], 'frac', d['roofline']['frac'])"; done

