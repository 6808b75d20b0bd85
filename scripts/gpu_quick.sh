# Quick iteration: encoder + attention GPU tests and the default bench line.
set -x
OUT=${OUT:-gpurun_out/quick}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_encoder.py tests/test_gpu_attention.py tests/test_gpu_kernels.py -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 600 python bench.py --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err
