# q64 backward clusters of 4 (Q / dO quarters multicast to all four; abtest/libupipe_q4.so) vs pairs (in-tree)
set -x
UPIPE_LIB=abtest/libupipe_q4.so timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu -k "bwd and not subprocess" -p no:cacheprovider -x 2>&1 | tail -2
UPIPE_LIB=abtest/libupipe_q4.so timeout 900 python -m pytest tests/test_gpu_layer.py -q -m gpu -k "not deterministic" -p no:cacheprovider -x 2>&1 | tail -2
for i in 1 2; do
  UPIPE_LIB=abtest/libupipe_q4.so timeout 300 python profiles/attn_shapes.py --reps 3 131072:8:2 131072:1:1 2>&1 | sed "s/^/[q4] /"
  timeout 300 python profiles/attn_shapes.py --reps 3 131072:8:2 131072:1:1 2>&1 | sed "s/^/[new] /"
done
for i in 1 2; do
  UPIPE_LIB=abtest/libupipe_q4.so timeout 600 python bench.py --quick --steps 4 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('[q4] bench', round(d['value']), d['phase_ms_per_step'], d['clocks']['sm_mhz'])"
  timeout 600 python bench.py --quick --steps 4 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('[new] bench', round(d['value']), d['phase_ms_per_step'], d['clocks']['sm_mhz'])"
done
