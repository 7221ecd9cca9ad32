# 32B-class layer (64 Q / 8 KV heads, d 128, hidden 5120; BASELINE configs[4] at CP 1) at 128K and 1M, with the Ulysses comparison
timeout 900 python bench.py --model 32b --no-cpu-baseline > gpurun_out/bench_32b_128k.json 2> gpurun_out/bench_32b_128k.err; echo rc=$?
timeout 2400 python bench.py --model 32b --seq 1048576 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_32b_1m.json 2> gpurun_out/bench_32b_1m.err; echo rc=$?
