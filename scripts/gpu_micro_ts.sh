nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Ipaper_2602_21196_b200/csrc profiles/micro_mma.cu -o /tmp/micro_mma && timeout 120 /tmp/micro_mma
