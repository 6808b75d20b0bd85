# Round profile: GPU tests, smoke, bench lines (documents, passages, varlen, reference arm),
# window sweep, launch list, ncu --set full of the top kernels.  Outputs in gpurun_out/round/.
set -x
OUT=${OUT:-gpurun_out/round2}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $OUT/smi.txt
# (GPU tests run separately this round)
# (smoke run separately)
timeout 900 python bench.py > $OUT/bench_n1.json 2> $OUT/bench_n1.err
timeout 600 python bench.py --impl reference > $OUT/bench_reference_n1.json 2> $OUT/bench_reference_n1.err
timeout 600 python bench.py --doc-len 164 --pairs-per-gpu 1024 --no-cpu-baseline > $OUT/bench_passages_n1.json 2> $OUT/bench_passages.err
timeout 600 python bench.py --varlen --no-cpu-baseline > $OUT/bench_varlen_n1.json 2> $OUT/bench_varlen.err
timeout 600 python scripts/rerank_c5.py --queries 50 --run-file $OUT/c5_run_q50.txt > $OUT/rerank_c5_n1.json 2> $OUT/rerank_c5.err
timeout 600 python scripts/rerank_c5.py --queries 50 --prune-last-layer >> $OUT/rerank_c5_n1.json 2>> $OUT/rerank_c5.err
timeout 600 python scripts/attn_sweep.py --windows 1,4,16,32,64,128,256,inf > $OUT/sweep.jsonl 2>&1
timeout 300 python scripts/attn_sweep.py --windows 4,64 --patterns qds >> $OUT/sweep.jsonl 2>&1
timeout 300 python scripts/attn_sweep.py --windows inf --patterns full,longformer >> $OUT/sweep.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-variants > $OUT/ncu_launches.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:band_attn -c 1 -o $OUT/band_w4 python scripts/attn_sweep.py --windows 4 --iters 1 > $OUT/ncu_band.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_attn -c 1 -o $OUT/tc_w256 python scripts/attn_sweep.py --windows 256 --iters 1 > $OUT/ncu_tc.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_attn -c 1 -o $OUT/tc_full python scripts/attn_sweep.py --windows inf --patterns full --iters 1 >> $OUT/ncu_tc.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"gemm_bias_gelu|residual_ln" -s 30 -c 2 -o $OUT/elt python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_elt.log 2>&1
ls -la $OUT
# round 2: the tcgen05 regime at every C4 window (w = 64, 256, sparse inf, full) + raw/source exports
for spec in "64 sparse" "256 sparse" "inf sparse" "inf full"; do
  set -- $spec
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_attn -c 1 -o $OUT/tc_$2_w$1 python scripts/attn_sweep.py --windows $1 --patterns $2 --iters 1 >> $OUT/ncu_tc.log 2>&1
  ncu -i $OUT/tc_$2_w$1.ncu-rep --page raw --csv > $OUT/tc_$2_w$1_raw.csv 2>/dev/null
done
ncu -i $OUT/band_w4.ncu-rep --page raw --csv > $OUT/band_w4_raw.csv 2>/dev/null
ncu -i $OUT/elt.ncu-rep --page raw --csv > $OUT/elt_raw.csv 2>/dev/null
rm -f $OUT/tc_w256.ncu-rep $OUT/tc_full.ncu-rep
ls -la $OUT
