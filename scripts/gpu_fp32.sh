#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_headline.py tests/test_gpu_encoder.py tests/test_gpu_kernels.py -x -q -p no:cacheprovider -k "split or x6 or f16 or fp32 or f32 or headline or layernorm" > gpurun_out/fp32_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/fp32_tests.log; tail -3 gpurun_out/fp32_tests.log
timeout 600 python scripts/probe/fp32_bench.py 5 2>&1 | tail -3
timeout 300 python scripts/probe/fp32_profile.py f16x3 > gpurun_out/fp32_prof.log 2>&1
grep -E "nvjet|split|band|residual|generic|Self CUDA time" gpurun_out/fp32_prof.log | awk '{print $1, $(NF-4), $(NF-3), $NF}' | head -20
