set -x
UPIPE_TRACE_LABELS=1 timeout 600 python bench.py --quick --steps 2 > gpurun_out/bench_lg.json 2> gpurun_out/bench_lg.err; echo $?; grep -E "trace\]" gpurun_out/bench_lg.err; tail -3 gpurun_out/bench_lg.err
UPIPE_PARITY_REPORT=gpurun_out/parity_r02.json timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "pytest exit $?"; tail -8 gpurun_out/gputest.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench $?; python -c "import json; d=json.loads(open('gpurun_out/bench.json').readlines()[-1]); print(d['value'], d['phase_ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['clocks'], d['peak_activation_gib'], d['ulysses'])"
