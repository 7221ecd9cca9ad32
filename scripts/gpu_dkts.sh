# dK MMA with dS^T from TMEM (UPIPE_BWD_DK_TS=1, in-tree build) vs shared memory (abtest/libupipe_ss.so)
set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py -q -m gpu -k "bwd or layer" -p no:cacheprovider -x 2>&1 | tail -3
B=ss bash scripts/ab_bwd.sh
