# bench variants of the round: Qwen3-32B-shaped layer (64 Q / 8 KV, D 5120) with and without the q/k norm + RoPE,
# and the GEMM phase by step label
set -x
timeout 900 python bench.py --model 32b --no-e2e --no-cpu-baseline > gpurun_out/bench_32b.json 2> gpurun_out/bench_32b.err; echo $?; tail -1 gpurun_out/bench_32b.json | cut -c1-600
timeout 900 python bench.py --model 32b --qk-norm 1e-6 --rope-base 1000000 --no-e2e --no-cpu-baseline > gpurun_out/bench_32b_qwen3.json 2> gpurun_out/bench_32b_qwen3.err; echo $?; tail -1 gpurun_out/bench_32b_qwen3.json | cut -c1-600
UPIPE_TRACE_LABELS=1 timeout 600 python bench.py --quick --steps 2 > gpurun_out/bench_labels.json 2> gpurun_out/bench_labels.err; echo $?; tail -40 gpurun_out/bench_labels.err
