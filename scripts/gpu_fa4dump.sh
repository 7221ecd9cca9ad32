mkdir -p gpurun_out/fa4dump
export CUTE_DSL_KEEP=ptx CUTE_DSL_DUMP_DIR=$PWD/gpurun_out/fa4dump
timeout 600 python profiles/fa4_compare.py --two-cta on --reps 1 8192:8:2 2>&1 | grep -v -i warn
ls -la gpurun_out/fa4dump | head
