#!/bin/bash
# Long documents: head-row pass warps per CTA x key splits (SC_BWD_HEAD_WARPS, SC_BWD_HEAD_KS).
mkdir -p gpurun_out
for hw in 1 2 8; do
  for ks in 4 8; do
    tag=hs_hw${hw}_ks${ks}
    SC_BWD_HEAD_WARPS=$hw SC_BWD_HEAD_KS=$ks timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none \
      --csv -k regex:head_ --log-file gpurun_out/$tag.csv python scripts/attn_bwd_prof.py --iters 1 > /dev/null 2>&1
    echo "== hw=$hw ks=$ks"; python scripts/ncu_csv_summary.py gpurun_out/$tag.csv | tail -n +2
  done
done
