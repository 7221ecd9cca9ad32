# one gpurun call: GPU tests (+ achieved-error report), kernel shapes, backward timeline, bench
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
UPIPE_PARITY_REPORT=gpurun_out/parity_r02.json timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider ${PYTEST_ARGS} > gpurun_out/gputest.log 2>&1; echo "pytest exit $?"; tail -15 gpurun_out/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
UPIPE_BWD_TIMELINE=1 timeout 600 python profiles/attn_shapes.py --reps 1 131072:8:2 131072:1:1 > gpurun_out/bwd_timeline.txt 2>&1; tail -6 gpurun_out/bwd_timeline.txt
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench $?; tail -2 gpurun_out/bench.json; tail -3 gpurun_out/bench.err
