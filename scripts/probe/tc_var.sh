#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
SC_TC_VARIANT=4 timeout 600 python -m pytest tests/test_gpu_attention.py -x -q -p no:cacheprovider -k "tcgen05 or full_size or packed" 2>&1 | tail -1
for v in -1 4; do
  echo "variant=$v"
  SC_TC_VARIANT=$v SWEEP_TC_ONLY=1 timeout 300 python scripts/sweep_quick.py > gpurun_out/tcv_$v.jsonl 2>&1
  python scripts/show_sweep.py gpurun_out/tcv_$v.jsonl | grep -v "=="
done
