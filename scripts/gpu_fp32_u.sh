#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for u in 1 2 4; do
  SC_SPLIT_GELU_U=$u timeout 300 python scripts/probe/fp32_profile.py f16x3 > gpurun_out/fp32_prof_u$u.log 2>&1
  echo "U=$u"; grep -E "split2h|Self CUDA time" gpurun_out/fp32_prof_u$u.log | awk '{print $2, $(NF-4), $NF}'
done
SC_SPLIT_GELU_U=2 timeout 600 python scripts/probe/fp32_bench.py 5 2>&1 | head -1
