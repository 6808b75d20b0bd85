#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_encoder.py -x -q -p no:cacheprovider 2>&1 | tail -3
for ipc in 1 2 3 4; do
  echo "ipc=$ipc"
  SC_TC_IPC=$ipc SWEEP_TC_ONLY=1 timeout 300 python scripts/sweep_quick.py > gpurun_out/tcs_$ipc.jsonl 2>&1
  python scripts/show_sweep.py gpurun_out/tcs_$ipc.jsonl | grep -v "=="
done
