# Band-kernel iteration: attention GPU tests, w sweep, one ncu --set full capture.
set -x
OUT=${OUT:-gpurun_out/band}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_kernels.py -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 300 python scripts/attn_sweep.py --windows 1,4,16,32,40,48,64 --algo band > $OUT/sweep.jsonl 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:band_attn -c 1 -o $OUT/band_full python scripts/attn_sweep.py --windows 4 --iters 1 > $OUT/ncu_band.log 2>&1
