set -x
timeout 300 python -m pytest tests/test_gpu_bench.py -q -m gpu -p no:cacheprovider -x 2>&1 | tail -2
for i in 1 2; do timeout 900 python bench.py --no-ulysses --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('bench', round(d['value']), 'e2e', round(d['e2e']['value']), d['clocks']['sm_mhz'])"; done
