#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_encoder.py -x -q -p no:cacheprovider 2>&1 | tail -1
for rep in 1 2; do
for q in 0 1; do
  echo "QFG=$q"
  SC_BAND_QFG=$q timeout 300 python scripts/attn_sweep.py --windows 4,9,12,16 > gpurun_out/qfg_$q.jsonl 2>&1
  grep -o '"w": "[0-9]*".*"us_per_seq_layer": [0-9.]*' gpurun_out/qfg_$q.jsonl | sed 's/"ms.*frac_hbm"/ frac/'
done
done
