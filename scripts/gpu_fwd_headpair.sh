# forward clusters of two query heads of one KV group (UPIPE_FWD_PAIR=2) vs query-tile pairs (default)
set -x
UPIPE_FWD_PAIR=2 timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu -k "fwd" -p no:cacheprovider -x 2>&1 | tail -2
UPIPE_FWD_PAIR=2 timeout 900 python -m pytest tests/test_gpu_layer.py -q -m gpu -k "not deterministic" -p no:cacheprovider -x 2>&1 | tail -2
for i in 1 2; do
  for E in "UPIPE_FWD_PAIR=2" "UPIPE_FWD_X=0"; do
    env $E timeout 300 python profiles/attn_shapes.py --reps 3 131072:8:2 131072:4:1 131072:2:1 2>&1 | sed "s/^/[$E] /"
  done
done
for i in 1 2; do
  for E in "UPIPE_FWD_PAIR=2" "UPIPE_FWD_X=0"; do
    env $E timeout 600 python bench.py --quick --steps 4 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('[$E] bench', round(d['value']), d['phase_ms_per_step'], d['clocks']['sm_mhz'])"
  done
done
