# forward exp split: 1 in 6 / 12 / 16 (abtest) vs 1 in 8 (in-tree)
for i in 1 2; do
  for B in p6 p12 p16 new; do
    L=""; [ $B != new ] && L="UPIPE_LIB=abtest/libupipe_$B.so"
    env $L timeout 300 python profiles/attn_shapes.py --reps 3 131072:8:2 2>&1 | sed "s/^/[$B] /"
  done
done
for i in 1 2; do
  for B in p6 p12 p16 new; do
    L=""; [ $B != new ] && L="UPIPE_LIB=abtest/libupipe_$B.so"
    env $L timeout 600 python bench.py --quick --steps 4 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('[$B] bench', round(d['value']), d['phase_ms_per_step'], d['clocks']['sm_mhz'])"
  done
done
