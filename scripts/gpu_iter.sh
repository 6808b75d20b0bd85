#!/bin/bash
# Iteration check: attention/encoder GPU tests, then the headline bench (no variants) twice + the quick sweep.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_encoder.py tests/test_gpu_headline.py -x -q -p no:cacheprovider ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/iter_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/iter_tests.log
tail -3 gpurun_out/iter_tests.log
for rep in 1 2; do
  timeout 300 python bench.py --no-variants --no-cpu-baseline --steps 10 > gpurun_out/iter_bench$rep.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/iter_bench$rep.json')); r=d['roofline']
print('bench', round(d['value'],1), 'instep', round(r['frac'],4), round(r['avg_launch_ms']*1e3,1), 'us  alone', round(r['standalone']['frac'],4), round(r['standalone']['median_ms']*1e3,1), 'us', d['clocks']['sm_mhz'], d['parity']['max_abs_err'])"
done
timeout 300 python scripts/sweep_quick.py > gpurun_out/iter_sweep.jsonl 2>&1
python scripts/show_sweep.py gpurun_out/iter_sweep.jsonl 2>/dev/null | head -8
