# final check at HEAD: full GPU suite, smoke, default bench line
set -x
timeout 2700 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/gputest_c.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/gputest_c.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_c.json 2> gpurun_out/bench_c.err; echo bench $?; python -c "import json; d=json.loads(open('gpurun_out/bench_c.json').readlines()[-1]); print(d['value'], d['phase_ms_per_step'], d['roofline']['frac'], d['roofline']['achieved'], d['e2e']['value'], d['clocks'], d['peak_activation_gib'], d['ulysses']['upipe_over_ulysses'])"
