# cta_group::2 attention backward (UPIPE_BWD_CTA2=1): kernel parity, then timing next to the default kernel
set -x
export UPIPE_BWD_CTA2=1
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -m gpu -k "attn_bwd and not dim_major and not deterministic and not subprocess" -p no:cacheprovider -x 2>&1 | tail -3
timeout 300 python profiles/attn_shapes.py --reps 3 32768:8:2 131072:8:2 131072:1:1
UPIPE_BWD_CTA2=0 timeout 300 python profiles/attn_shapes.py --reps 3 32768:8:2 131072:8:2 131072:1:1
