#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
SC_BAND_GROUPS=1 timeout 300 python -m pytest tests/test_gpu_attention.py tests/test_gpu_encoder.py tests/test_gpu_headline.py -x -q -p no:cacheprovider 2>&1 | tail -1
for rep in 1 2; do
for gr in 0 1; do
  SC_BAND_GROUPS=$gr timeout 300 python scripts/attn_sweep.py --windows 1,4 > gpurun_out/grp_$gr.jsonl 2>&1
  SC_BAND_GROUPS=$gr timeout 300 python bench.py --no-variants --no-cpu-baseline --steps 10 > gpurun_out/grpb_$gr.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/grpb_$gr.json')); r=d['roofline']
sw=[json.loads(l) for l in open('gpurun_out/grp_$gr.jsonl') if l.startswith('{')]
print('groups=$gr', [(x['w'], x['us_per_seq_layer']) for x in sw], 'bench', round(d['value'],1), 'instep', round(r['frac'],4), 'alone', round(r['standalone']['frac'],4), d['clocks']['sm_mhz'])"
done
done
