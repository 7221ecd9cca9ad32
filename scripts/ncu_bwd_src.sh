# ncu --set full with source of the attention backward (q64) at S = 32K, 8 q / 2 kv heads (the bench's launch shape)
set -x
timeout 900 ncu --set full --import-source on --clock-control none -k regex:attn_bwd_q64 -c 1 -f -o gpurun_out/bwd_q64_32k python profiles/attn_shapes.py --reps 1 32768:8:2 > gpurun_out/ncu_bwd.log 2>&1; echo ncu $?
tail -3 gpurun_out/ncu_bwd.log
