#!/bin/bash
# Experiment: QKV GEMM + attention per chunk of sequences (q|k|v L2-resident) vs the whole batch.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for cfg in "0 0" "0 1" "4 1" "5 1" "6 1" "8 1" "5 0"; do
  set -- $cfg
  SC_QKV_CHUNK=$1 SC_BAND_ITEMS=$2 timeout 300 python bench.py --no-variants --no-cpu-baseline --steps 10 > gpurun_out/chunk_$1_$2.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/chunk_$1_$2.json')); print('chunk=$1 items=$2', round(d['value'],1), round(d['ms_per_step'],2), d['parity']['max_abs_err'], d['clocks']['sm_mhz'])"
done
