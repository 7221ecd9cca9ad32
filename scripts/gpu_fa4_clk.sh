timeout 900 python profiles/fa4_compare.py --two-cta both --ours --reps 5 131072:8:2 2>&1 | grep -v -i warn
