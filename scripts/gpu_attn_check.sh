#!/bin/bash
# attention parity tests + C4 sweep + launch list at w=64 (round-2 tc kernel work)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_encoder.py -x -q -p no:cacheprovider > gpurun_out/attn_tests.log 2>&1
echo "rc=$?" >> gpurun_out/attn_tests.log
timeout 300 python scripts/sweep_quick.py > gpurun_out/sweep.jsonl 2>&1
for w in 64 256; do
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/attn_w$w.csv python scripts/attn_one.py --w $w --iters 2 > /dev/null 2>&1
done
