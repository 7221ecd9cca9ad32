# GEMM pair MMAs issued by a lane elected once (in-tree) vs elect.sync in every MMA asm (abtest/libupipe_gw.so)
set -x
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu -k "gemm" -p no:cacheprovider -x 2>&1 | tail -2
for i in 1 2; do
  UPIPE_LIB=abtest/libupipe_gw.so timeout 300 python profiles/gemm_time.py 2>&1 | sed "s/^/[gw] /"
  timeout 300 python profiles/gemm_time.py 2>&1 | sed "s/^/[new] /"
done
for i in 1 2; do
  UPIPE_LIB=abtest/libupipe_gw.so timeout 600 python bench.py --quick --steps 4 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('[gw] bench', round(d['value']), d['phase_ms_per_step'], d['clocks']['sm_mhz'])"
  timeout 600 python bench.py --quick --steps 4 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('[new] bench', round(d['value']), d['phase_ms_per_step'], d['clocks']['sm_mhz'])"
done
