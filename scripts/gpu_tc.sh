# tcgen05-kernel iteration: attention GPU tests, wide-window sweep, ncu --set full of tc_attn_kernel.
set -x
OUT=${OUT:-gpurun_out/tc}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_attention.py -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 300 python scripts/attn_sweep.py --windows 64,128,256,inf > $OUT/sweep.jsonl 2>&1
timeout 300 python scripts/attn_sweep.py --windows inf --patterns full >> $OUT/sweep.jsonl 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_attn -c 1 -o $OUT/tc_full_inf python scripts/attn_sweep.py --windows inf --patterns full --iters 1 > $OUT/ncu_tc.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_attn -c 1 -o $OUT/tc_full_w256 python scripts/attn_sweep.py --windows 256 --iters 1 >> $OUT/ncu_tc.log 2>&1
