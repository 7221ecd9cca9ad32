# same-box A/B of an env switch: ENVA vs ENVB, alternating, bench --quick with step labels
set -x
for i in 1 2; do
  for E in "$ENVA" "$ENVB"; do
    env $E UPIPE_TRACE_LABELS=1 timeout 600 python bench.py --quick --steps 2 > gpurun_out/ab.json 2> gpurun_out/ab.err
    echo "== $E"; grep -E "trace\] (${LABELS:-dO})" gpurun_out/ab.err; python -c "import json; d=json.loads(open('gpurun_out/ab.json').readlines()[-1]); print(round(d['value']), d['phase_ms_per_step'], d['clocks']['sm_mhz'])"
  done
done
