#!/bin/bash
# Round-2 first GPU pass: new parity tests + a bench line.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 900 python -m pytest tests/test_gpu_headline.py tests/test_gpu_rerank.py tests/test_gpu_kernels.py tests/test_gpu_encoder.py \
  -k "headline or rerank or split or x6 or golden or nonfinite or world2" -q -s -p no:cacheprovider > gpurun_out/t1.log 2>&1
echo "pytest rc=$?" >> gpurun_out/t1.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench1.json 2> gpurun_out/bench1.err
echo "bench rc=$?" >> gpurun_out/bench1.err
