# q64 backward visiting order: heads inner (abtest/libupipe_hi.so) vs heads outer (in-tree default)
set -x
UPIPE_LIB=abtest/libupipe_hi.so timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu -k "bwd and not subprocess" -p no:cacheprovider -x 2>&1 | tail -2
for i in 1 2; do
  UPIPE_LIB=abtest/libupipe_hi.so timeout 300 python profiles/attn_shapes.py --reps 3 131072:8:2 131072:1:1 2>&1 | sed "s/^/[hi] /"
  timeout 300 python profiles/attn_shapes.py --reps 3 131072:8:2 131072:1:1 2>&1 | sed "s/^/[new] /"
done
for i in 1 2; do
  UPIPE_LIB=abtest/libupipe_hi.so timeout 600 python bench.py --quick --steps 4 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('[hi] bench', round(d['value']), d['phase_ms_per_step'], d['clocks']['sm_mhz'])"
  timeout 600 python bench.py --quick --steps 4 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('[new] bench', round(d['value']), d['phase_ms_per_step'], d['clocks']['sm_mhz'])"
done
for B in hi new; do
  L=""; [ $B != new ] && L="UPIPE_LIB=abtest/libupipe_$B.so"
  env $L timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none -k regex:attn_bwd_q64 -c 1 --csv python profiles/attn_shapes.py --reps 1 131072:8:2 2>/dev/null | grep -E "dram__|gpu__time|lts__t_bytes" | sed "s/^/[$B] /"
done
