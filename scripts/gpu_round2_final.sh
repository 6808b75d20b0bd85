#!/bin/bash
# Round-2 final profile with the final kernels: bench arms, passages / varlen / C5 lines, sweep,
# headline-step launch list, ncu --set full of the attention kernels + the elementwise passes,
# summarised on the box (scripts/summarize_profiles.py) so only summaries travel back.
cd "$GRAFT_REPO_ROOT"
OUT=${OUT:-gpurun_out/round2f}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $OUT/smi.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke.txt 2>&1
timeout 900 python bench.py > $OUT/bench_n1.json 2> $OUT/bench_n1.err
timeout 600 python bench.py --impl reference > $OUT/bench_reference_n1.json 2> $OUT/bench_reference_n1.err
timeout 600 python bench.py --doc-len 164 --pairs-per-gpu 1024 --no-cpu-baseline > $OUT/bench_passages_n1.json 2> $OUT/bench_passages.err
timeout 600 python bench.py --varlen --no-cpu-baseline > $OUT/bench_varlen_n1.json 2> $OUT/bench_varlen.err
timeout 600 python scripts/rerank_c5.py --queries 50 --run-file $OUT/c5_run_q50.txt > $OUT/rerank_c5_n1.json 2> $OUT/rerank_c5.err
timeout 600 python scripts/rerank_c5.py --queries 50 --prune-last-layer >> $OUT/rerank_c5_n1.json 2>> $OUT/rerank_c5.err
timeout 600 python scripts/attn_sweep.py --windows 1,4,16,32,40,48,64,128,256,inf > $OUT/sweep.jsonl 2>&1
timeout 300 python scripts/attn_sweep.py --windows 4,64 --patterns qds >> $OUT/sweep.jsonl 2>&1
timeout 300 python scripts/attn_sweep.py --windows inf --patterns full,longformer >> $OUT/sweep.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-variants > $OUT/ncu_launches.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:band_attn -c 1 -o $OUT/band_w4 python scripts/attn_sweep.py --windows 4 --iters 1 > $OUT/ncu_band.log 2>&1
for spec in "64 sparse" "256 sparse" "inf sparse" "inf full"; do
  set -- $spec
  timeout 600 ncu --set full --clock-control none -k regex:tc_attn -c 1 -o $OUT/tc_$2_w$1 python scripts/attn_sweep.py --windows $1 --patterns $2 --iters 1 >> $OUT/ncu_tc.log 2>&1
done
timeout 600 ncu --set full --clock-control none -k regex:"gemm_bias_gelu|residual_ln|merge_full" -s 30 -c 3 -o $OUT/elt python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-variants > $OUT/ncu_elt.log 2>&1
ncu -i $OUT/band_w4.ncu-rep --page source --csv --print-source sass > $OUT/band_w4_sass.csv 2>/dev/null
ncu -i $OUT/band_w4.ncu-rep --page raw --csv > $OUT/band_w4_raw.csv 2>/dev/null
python scripts/summarize_profiles.py $OUT $OUT/summary > $OUT/summary.log 2>&1
rm -f $OUT/tc_*.ncu-rep $OUT/elt.ncu-rep
ls -la $OUT $OUT/summary
