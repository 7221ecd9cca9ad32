set -x
UPIPE_TRACE_LABELS=1 timeout 600 python bench.py --quick --steps 2 > gpurun_out/bench_labels2.json 2> gpurun_out/bench_labels2.err; echo $?; grep -E "dW|dX|proj|dO|out" gpurun_out/bench_labels2.err
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -x > gpurun_out/gputest.log 2>&1; echo "pytest exit $?"; tail -5 gpurun_out/gputest.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench $?; tail -1 gpurun_out/bench.json | cut -c1-300; python -c "import json; d=json.loads(open('gpurun_out/bench.json').readlines()[-1]); print(d['phase_ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['clocks'])"
