# U ablation at 128K on one GPU at HEAD: U = 8 / 16 / 32 (Ulysses) and U = 8 with the naive per-stage K/V schedule
for a in "--chunk 8" "--chunk 16" "--chunk 32" "--chunk 8 --naive-kv"; do
  timeout 900 python bench.py $a --no-ulysses --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.readline()); c=d['config']
print(json.dumps({'args': '$a', 'tokens_per_s': round(d['value']), 'ms_per_step': round(d['ms_per_step'],1), 'phase_ms_per_step': {k: round(v,1) for k,v in d['phase_ms_per_step'].items()}, 'peak_activation_gib': round(d['peak_activation_gib'],2), 'workspace_gib': round(d['workspace_gib'],2), 'chunk_buffers_gib': round(d['chunk_buffers_gib'],2), 'sm_mhz': d['clocks']['sm_mhz']}))"
done
