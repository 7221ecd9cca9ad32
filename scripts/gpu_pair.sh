set -x
UPIPE_BWD_PAIR=1 timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu -k "bwd and not subprocess" -p no:cacheprovider -x 2>&1 | tail -5
UPIPE_BWD_PAIR=1 timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_fullsize.py -q -m gpu -k "not deterministic" -p no:cacheprovider -x 2>&1 | tail -5
for i in 1 2; do
  UPIPE_BWD_PAIR=1 timeout 300 python profiles/attn_shapes.py --reps 3 131072:8:2 131072:1:1 2>&1 | sed "s/^/[pair] /"
  timeout 300 python profiles/attn_shapes.py --reps 3 131072:8:2 131072:1:1 2>&1 | sed "s/^/[base] /"
done
for i in 1 2; do
  UPIPE_BWD_PAIR=1 timeout 600 python bench.py --quick --steps 4 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('[pair] bench', round(d['value']), d['phase_ms_per_step'], d['clocks']['sm_mhz'])"
  timeout 600 python bench.py --quick --steps 4 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('[base] bench', round(d['value']), d['phase_ms_per_step'], d['clocks']['sm_mhz'])"
done
