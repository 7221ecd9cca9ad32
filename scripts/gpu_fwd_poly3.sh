# forward exp split: 1 in 8 on the FMA pipe (in-tree) vs 1 in 4 (abtest/libupipe_p4.so), plus forward parity
set -x
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu -k "fwd" -p no:cacheprovider -x 2>&1 | tail -2
timeout 600 python -m pytest tests/test_gpu_layer.py -q -m gpu -k "not deterministic" -p no:cacheprovider -x 2>&1 | tail -2
for i in 1 2 3; do
  for B in p4 new; do
    L=""; [ $B != new ] && L="UPIPE_LIB=abtest/libupipe_$B.so"
    env $L timeout 300 python profiles/attn_shapes.py --reps 3 131072:8:2 131072:1:1 2>&1 | sed "s/^/[$B] /"
  done
done
for i in 1 2 3; do
  for B in p4 new; do
    L=""; [ $B != new ] && L="UPIPE_LIB=abtest/libupipe_$B.so"
    env $L timeout 600 python bench.py --quick --steps 4 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('[$B] bench', round(d['value']), d['phase_ms_per_step'], d['clocks']['sm_mhz'])"
  done
done
