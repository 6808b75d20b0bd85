# Kernel tests + three default bench lines (noise estimate).
set -x
OUT=${OUT:-gpurun_out/b3}
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_encoder.py -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for rep in 1 2 3; do
  timeout 600 python bench.py --no-cpu-baseline --steps 20 > $OUT/bench_$rep.json 2> $OUT/bench_$rep.err
done
