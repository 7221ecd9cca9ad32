# cta_group::2 MMA rates and the M = 128 pair accumulator layout; FlashAttention-4 (library, context) vs ours
set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Ipaper_2602_21196_b200/csrc profiles/micro_pair.cu -o /tmp/micro_pair && timeout 120 /tmp/micro_pair
timeout 900 python profiles/fa4_compare.py --two-cta both 32768:8:2 131072:8:2 131072:1:1 2>&1 | grep -v -i warn
