#!/bin/bash
# A/B of the head-row pass warps per CTA (SC_BWD_HEAD_WARPS) on the passage and long-document shapes.
mkdir -p gpurun_out
for hw in 0 1 2; do
  for cfg in "--nseq 64 --doc-len 164" "--nseq 8 --doc-len 4086"; do
    tag=hw${hw}_$(echo $cfg | tr -d ' -')
    SC_BWD_HEAD_WARPS=$hw timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      -k regex:head_ --log-file gpurun_out/$tag.csv python scripts/attn_bwd_prof.py $cfg --iters 1 > /dev/null 2>&1
    python scripts/ncu_csv_summary.py gpurun_out/$tag.csv
  done
done
