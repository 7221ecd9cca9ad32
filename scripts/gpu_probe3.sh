set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Ipaper_2602_21196_b200/csrc profiles/micro_pair.cu -o /tmp/micro_pair
timeout 120 /tmp/micro_pair 2>&1 | grep -v "probe\|lane"
SMEM_KB=200 timeout 120 /tmp/micro_pair 2>&1 | grep -v "probe\|lane"
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv
