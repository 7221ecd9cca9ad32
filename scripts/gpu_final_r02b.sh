# end of round 2: full GPU suite, smoke, bench, launch list, ncu --set full of the (now CTA-pair) forward
set -x
UPIPE_PARITY_REPORT=gpurun_out/parity_r02b.json timeout 2700 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "pytest exit $?"; tail -6 gpurun_out/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench $?; python -c "import json; d=json.loads(open('gpurun_out/bench.json').readlines()[-1]); print(d['value'], d['phase_ms_per_step'], d['roofline']['frac'], d['roofline']['achieved'], d['e2e']['value'], d['clocks'], d['peak_activation_gib'], d['ulysses']['upipe_over_ulysses'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r02_launches_fwdpair.csv python bench.py --quick --steps 1 --warmup 1 > /dev/null 2>&1; echo launches $?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:attn_fwd -c 1 -f -o gpurun_out/r02_fwd_pair_128k python bench.py --quick --steps 1 --warmup 1 > gpurun_out/ncu_fwd_pair.log 2>&1; echo ncu_fwd $?
