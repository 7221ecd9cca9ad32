set -x
timeout 1200 python -m pytest tests/test_gpu_bench.py -q -m gpu -k multi_rank -p no:cacheprovider > gpurun_out/gpubench.log 2>&1; echo "pytest exit $?"; tail -15 gpurun_out/gpubench.log
timeout 1500 python bench.py --seq 1048576 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_1m.json 2> gpurun_out/bench_1m.err; echo $?; python -c "import json; d=json.loads(open('gpurun_out/bench_1m.json').readlines()[-1]); print(d['value'], d['ms_per_step'], d['phase_ms_per_step'], d['roofline']['frac'], d['clocks'], d['peak_activation_gib'], d.get('ulysses'), d.get('e2e',{}).get('value'))"
