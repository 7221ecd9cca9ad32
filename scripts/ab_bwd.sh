# A/B of a backward-kernel variant: abtest/libupipe_<B>.so vs the in-tree build, same box, alternating
set -x
B=${B:-nopipe}
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu -k "bwd" -p no:cacheprovider 2>&1 | tail -2
for i in 1 2 3; do
  UPIPE_LIB=abtest/libupipe_$B.so timeout 300 python profiles/attn_shapes.py --reps 3 131072:8:2 131072:1:1 2>&1 | sed "s/^/[$B] /"
  timeout 300 python profiles/attn_shapes.py --reps 3 131072:8:2 131072:1:1 2>&1 | sed "s/^/[new] /"
done
for i in 1 2; do
  UPIPE_LIB=abtest/libupipe_$B.so timeout 600 python bench.py --quick --steps 4 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('[$B] bench', round(d['value']), d['phase_ms_per_step'], d['clocks']['sm_mhz'])"
  timeout 600 python bench.py --quick --steps 4 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('[new] bench', round(d['value']), d['phase_ms_per_step'], d['clocks']['sm_mhz'])"
done
