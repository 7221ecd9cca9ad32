# GEMM launch choices under the power cap (bench step, same box): default vs UPIPE_GEMM_PAIR=2 (two pairs share B) vs UPIPE_GEMM_WIDE=0
for i in 1 2 3; do
  for E in "UPIPE_X=0" "UPIPE_GEMM_PAIR=2" "UPIPE_GEMM_WIDE=0"; do
    env $E timeout 600 python bench.py --quick --steps 4 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('[$E] bench', round(d['value']), {k: round(v,2) for k,v in d['phase_ms_per_step'].items()}, d['clocks']['sm_mhz'])"
  done
done
