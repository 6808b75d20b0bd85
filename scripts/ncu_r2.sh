#!/bin/bash
# ncu --set full captures of the attention kernels (one launch each) + raw/source CSV exports.
# WINDOWS (default "4 64 256 inf"), KERNEL regex (default tc_attn_kernel|band_attn_kernel), EXTRA args for attn_one.py
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
TAG=${TAG:-r2}
for w in ${WINDOWS:-4 64 256 inf}; do
  ncu --set full --import-source on --clock-control none -k "regex:${KERNEL:-tc_attn_kernel|band_attn_kernel}" -c 1 -o /tmp/ncu_w$w \
    python scripts/attn_one.py --w $w --iters 1 ${EXTRA} > gpurun_out/ncu_${TAG}_w$w.log 2>&1
  ncu -i /tmp/ncu_w$w.ncu-rep --page raw --csv > gpurun_out/raw_${TAG}_w$w.csv 2>/dev/null
  ncu -i /tmp/ncu_w$w.ncu-rep --page source --csv --print-source sass > gpurun_out/sass_${TAG}_w$w.csv 2>/dev/null
done
