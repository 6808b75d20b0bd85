set -x
OUT=gpurun_out/tcp
mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_attn -c 1 -o $OUT/w256 python scripts/attn_sweep.py --windows 256 --iters 1 > $OUT/ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_attn -c 1 -o $OUT/inf python scripts/attn_sweep.py --windows inf --iters 1 >> $OUT/ncu.log 2>&1
