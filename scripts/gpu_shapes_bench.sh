set -x
timeout 900 python profiles/attn_shapes.py > gpurun_out/attn_shapes_full.jsonl 2>&1; cat gpurun_out/attn_shapes_full.jsonl
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench $?; python -c "import json; d=json.loads(open('gpurun_out/bench.json').readlines()[-1]); print(d['value'], d['phase_ms_per_step'], d['roofline'], d['e2e']['value'], d['clocks'], d['peak_activation_gib'], d['ulysses']['upipe_over_ulysses'])"
