# Encoder-loop iteration: all GPU tests, bench, launch list of one step, ncu of the elementwise kernels.
set -x
OUT=${OUT:-gpurun_out/e2e}
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q -rA > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 600 python bench.py --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"bias_gelu|residual_ln" -s 30 -c 2 -o $OUT/elt_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_elt.log 2>&1
