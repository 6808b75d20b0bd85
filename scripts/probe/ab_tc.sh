#!/bin/bash
# A/B two library builds on the tcgen05-regime sweep (+ the attention tests on the new one).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
SC_LIB_PATH=paper_2312_17649_b200/_lib_ab/new.so timeout 900 python -m pytest tests/test_gpu_attention.py -x -q -p no:cacheprovider 2>&1 | tail -2
for rep in 1 2; do
for L in old new; do
  echo "== $L (rep $rep)"
  SC_LIB_PATH=paper_2312_17649_b200/_lib_ab/$L.so SWEEP_TC_ONLY=1 timeout 300 python scripts/sweep_quick.py > gpurun_out/abtc_$L.jsonl 2>&1
  python scripts/show_sweep.py gpurun_out/abtc_$L.jsonl | grep -v "=="
done
done
