#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 300 python scripts/probe/sweep_context.py > gpurun_out/sweep_context.log 2>&1
timeout 300 python scripts/probe/fp32_profile.py f16x3 > gpurun_out/fp32_prof.log 2>&1
ncu --set full --import-source on --clock-control none -k "regex:band_attn_kernel" -c 1 -o gpurun_out/band_w4 \
    python scripts/attn_one.py --w 4 --iters 1 > gpurun_out/ncu_band.log 2>&1
ncu -i gpurun_out/band_w4.ncu-rep --page source --csv --print-source sass > gpurun_out/band_w4_sass.csv 2>/dev/null
ncu -i gpurun_out/band_w4.ncu-rep --page raw --csv > gpurun_out/band_w4_raw.csv 2>/dev/null
