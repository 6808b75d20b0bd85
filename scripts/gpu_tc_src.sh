#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for w in ${WINDOWS:-64}; do
ncu --set full --import-source on --clock-control none -k "regex:tc_attn_kernel" -c 1 -o gpurun_out/tc_w$w \
    python scripts/attn_one.py --w $w --iters 1 > gpurun_out/ncu_tc_w$w.log 2>&1
ncu -i gpurun_out/tc_w$w.ncu-rep --page source --csv --print-source sass > gpurun_out/tc_w${w}_sass.csv 2>/dev/null
ncu -i gpurun_out/tc_w$w.ncu-rep --page raw --csv > gpurun_out/tc_w${w}_raw.csv 2>/dev/null
done
