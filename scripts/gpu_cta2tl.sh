export UPIPE_BWD_CTA2=1 UPIPE_BWD_TIMELINE=1
timeout 300 python profiles/attn_shapes.py --reps 1 32768:8:2 2>&1 | tail -4
UPIPE_BWD_CTA2=0 timeout 300 python profiles/attn_shapes.py --reps 1 32768:8:2 2>&1 | tail -3
