# max-context probe on ONE B200: UPipe (U = 8) at 3M tokens (BASELINE configs[3] regime, which names 8 GPUs)
timeout 1700 python bench.py --seq 3145728 --steps 1 --warmup 1 --no-ulysses --no-e2e --no-cpu-baseline > gpurun_out/bench_3m.json 2> gpurun_out/bench_3m.err; echo rc=$?
tail -3 gpurun_out/bench_3m.err
