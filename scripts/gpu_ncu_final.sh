# ncu evidence at the final HEAD: launch list of one 128K bench step, --set full of the forward (1-in-8 exp split)
set -x
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r02_launches_final_e.csv python bench.py --quick --steps 1 --warmup 1 > /dev/null 2>&1; echo launches $?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:attn_fwd -c 1 -f -o gpurun_out/r02_fwd_final_128k python bench.py --quick --steps 1 --warmup 1 > gpurun_out/ncu_fwd_final.log 2>&1; echo ncu_fwd $?
