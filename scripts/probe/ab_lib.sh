#!/bin/bash
# A/B two builds of the library on one box: band/tc sweep + bench in-step roofline, alternating.
cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for L in ${LIBS:-old new}; do
  echo "== $L (rep $rep)"
  SC_LIB_PATH=paper_2312_17649_b200/_lib_ab/$L.so timeout 300 python scripts/sweep_quick.py > gpurun_out/ab_$L.jsonl 2>&1
  python scripts/show_sweep.py gpurun_out/ab_$L.jsonl 2>/dev/null | sed -n 2,4p
  SC_LIB_PATH=paper_2312_17649_b200/_lib_ab/$L.so timeout 600 python bench.py --no-variants --no-cpu-baseline --steps 10 > gpurun_out/ab_bench_$L.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ab_bench_$L.json')); print('bench', round(d['value'],1), round(d['roofline']['frac'],4), round(d['roofline']['standalone']['frac'],4), d['clocks']['sm_mhz'])"
done
done
