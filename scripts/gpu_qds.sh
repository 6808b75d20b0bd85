set -x
OUT=gpurun_out/qds
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_attention.py -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 300 python scripts/attn_sweep.py --windows 4,64 --patterns qds,longformer > $OUT/sweep.jsonl 2>&1
