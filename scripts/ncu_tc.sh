#!/bin/bash
# Full ncu capture of the tcgen05 attention kernel at several windows; raw + source pages as CSV.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for w in ${WINDOWS:-64 256 inf}; do
  ncu --set full --import-source on --clock-control none -k regex:${KERNEL:-tc_attn_kernel} -c 1 -o /tmp/tc_w$w \
    python scripts/attn_one.py --w $w --iters 1 ${EXTRA} > gpurun_out/ncu_w$w.log 2>&1
  ncu -i /tmp/tc_w$w.ncu-rep --page raw --csv > gpurun_out/tc_raw_w$w.csv 2>/dev/null
  ncu -i /tmp/tc_w$w.ncu-rep --page details --csv > gpurun_out/tc_details_w$w.csv 2>/dev/null
  ncu -i /tmp/tc_w$w.ncu-rep --page source --csv --print-source sass > gpurun_out/tc_sass_w$w.csv 2>/dev/null
done
