# Sweep the tcgen05 kernel variants (SC_TC_VARIANT) over wide windows; attention tests per variant.
set -x
OUT=gpurun_out/tcv
mkdir -p $OUT
for v in ${VARIANTS:-2 6 7 8}; do
  echo "variant=$v" >> $OUT/sweep.txt
  SC_TC_VARIANT=$v timeout 300 python scripts/attn_sweep.py --windows 16,32,64,256,inf --algo tc >> $OUT/sweep.txt 2>&1
  SC_TC_VARIANT=$v timeout 600 python -m pytest tests/test_gpu_attention.py -x -q > $OUT/pytest_$v.log 2>&1; echo "rc=$?" >> $OUT/pytest_$v.log
done
timeout 300 python scripts/attn_sweep.py --windows 16,32,48,64 --algo band > $OUT/band.txt 2>&1
