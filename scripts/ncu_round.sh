# ncu evidence of the round: launch list of one bench step, --set full of the dominant kernel (attn bwd) at the
# bench's launch shape, and the compute-sanitizer runs
set -x
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r02_launches_128k.csv python bench.py --quick --steps 1 --warmup 1 > /dev/null 2>&1; echo launches $?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:attn_bwd_q64 -c 1 -f -o gpurun_out/r02_bwd_q64_128k python bench.py --quick --steps 1 --warmup 1 > gpurun_out/ncu_bwd128k.log 2>&1; echo ncu_bwd $?
timeout 900 ncu --set full --clock-control none -k regex:attn_fwd -c 1 -f -o gpurun_out/r02_fwd_128k python bench.py --quick --steps 1 --warmup 1 > gpurun_out/ncu_fwd128k.log 2>&1; echo ncu_fwd $?
bash scripts/sanitize.sh
