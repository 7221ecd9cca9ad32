# BASELINE configs[2] at CP 1 on one GPU at the final HEAD: 1M tokens, UPipe U = 8 with the Ulysses comparison
timeout 3000 python bench.py --seq 1048576 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_1m_final.json 2> gpurun_out/bench_1m_final.err; echo rc=$?
