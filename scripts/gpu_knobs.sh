#!/bin/bash
# A/B of measurement knobs (env) on the headline bench: in-step / standalone roofline fractions.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
run() {
  local tag=$1; shift
  env "$@" timeout 300 python bench.py --no-variants --no-cpu-baseline --steps 10 > gpurun_out/knob_$tag.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/knob_$tag.json')); r=d['roofline']
print('$tag', round(d['value'],1), 'instep', round(r['frac'],4), round(r['avg_launch_ms']*1e3,1), 'us  alone', round(r['standalone']['frac'],4), round(r['standalone']['median_ms']*1e3,1), 'us', d['clocks']['sm_mhz'])" >> gpurun_out/knobs.txt
}
for rep in 1 2; do
  run base$rep X=1
  run clsskip$rep SC_BAND_CLS_SKIP=1
  run grid416_$rep SC_BAND_GRID=416
  run both$rep SC_BAND_CLS_SKIP=1 SC_BAND_GRID=416
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv python scripts/attn_one.py --w 4 --iters 2 > gpurun_out/attn_launches.csv 2>&1
