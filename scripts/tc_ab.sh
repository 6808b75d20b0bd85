#!/bin/bash
# tcgen05 attention: parity tests + C4 sweep per forced variant (SC_TC_VARIANT A/B).
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attention.py -x -q -p no:cacheprovider > gpurun_out/attn_tests.log 2>&1
echo "rc=$?" >> gpurun_out/attn_tests.log
timeout 300 python scripts/sweep_quick.py > gpurun_out/sweep_default.jsonl 2>&1
for v in ${VARIANTS:-4 5 1 0}; do
  SC_TC_VARIANT=$v timeout 300 python scripts/sweep_quick.py > gpurun_out/sweep_v$v.jsonl 2>&1
done
