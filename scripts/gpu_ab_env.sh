# A/B of an env switch on the bench line: VAR=<name>; runs bench with VAR=1 and VAR=0, twice each, alternating.
set -x
OUT=${OUT:-gpurun_out/ab}
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_attention.py -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for rep in 1 2; do
  for v in 1 0; do
    env $VAR=$v timeout 600 python bench.py --no-cpu-baseline --steps 20 > $OUT/bench_${v}_${rep}.json 2> $OUT/bench_${v}_${rep}.err
  done
done
