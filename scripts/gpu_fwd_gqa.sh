# forward at 128K: GQA 8/2 vs MHA 8/8 vs 1/1 (is the 8/2 gap to FA4 GQA-specific or the long run's clock?)
for i in 1 2; do
  timeout 300 python profiles/fa4_compare.py --two-cta off --ours --reps 3 131072:8:8 131072:8:2 131072:1:1 2>&1 | grep -v -i warn
done
