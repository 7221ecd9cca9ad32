# ncu --set full of the first dX GEMM of a bench step (gemm launch index 18 after the forward's Q, K|V, out proj)
set -x
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_kernel --launch-skip ${SKIP:-14} -c 4 -f -o gpurun_out/r02_gemm_bwd python bench.py --quick --steps 1 --warmup 1 > gpurun_out/ncu_gemm.log 2>&1; echo ncu $?; tail -3 gpurun_out/ncu_gemm.log
