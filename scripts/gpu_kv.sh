set -x
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -x -k "layout or kernels or ipc or rope or 32b or qk_norm or fullsize" > gpurun_out/gputest_kv.log 2>&1; echo "pytest exit $?"; tail -4 gpurun_out/gputest_kv.log
for r in 1 0 1 0; do
UPIPE_FUSED_ROWDOT=$r UPIPE_TRACE_LABELS=1 timeout 600 python bench.py --quick --steps 2 > gpurun_out/bench_l.json 2> gpurun_out/bench_l.err; echo "rowdot_fused=$r"; grep -E "trace\] (dO|rowdot|proj|dX|dW)" gpurun_out/bench_l.err; python -c "import json; d=json.loads(open('gpurun_out/bench_l.json').readlines()[-1]); print(round(d['value']), d['phase_ms_per_step'], d['clocks']['sm_mhz'])"
done
