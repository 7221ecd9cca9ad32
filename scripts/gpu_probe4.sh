nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Ipaper_2602_21196_b200/csrc profiles/micro_pair.cu -o /tmp/micro_pair; echo rc=$?
SMEM_KB=200 timeout 120 /tmp/micro_pair > /tmp/mp.out 2>&1; echo rc=$?
head -c 6000 /tmp/mp.out
