# forward CTA pairs on / off at the CP 8 per-rank shapes (4/1: U = 32, 2/1: U = 16) and 8/2, alternating
for i in 1 2 3; do
  for E in 1 0; do
    UPIPE_FWD_PAIR=$E timeout 300 python profiles/attn_shapes.py --reps 3 131072:4:1 131072:2:1 131072:8:2 2>&1 | sed "s/^/[pair=$E] /"
  done
done
