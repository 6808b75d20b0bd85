#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -s -p no:cacheprovider -k "x3h" 2>&1 | grep -E "fused max|passed|failed|Error|error" | head -10
timeout 900 python -m pytest tests/test_gpu_headline.py tests/test_gpu_encoder.py -x -q -p no:cacheprovider -k "split or x6 or f16 or fp32 or f32 or headline" 2>&1 | tail -2
timeout 600 python scripts/probe/fp32_bench.py 5 2>&1 | head -1
timeout 300 python scripts/probe/fp32_profile.py f16x3 > gpurun_out/fp32_prof.log 2>&1
grep -E "nvjet|split|band|residual|generic|gemm_x3h|Self CUDA time" gpurun_out/fp32_prof.log | awk '{print $1, $(NF-4), $NF}' | head -16
