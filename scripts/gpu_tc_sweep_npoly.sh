# Rebuild the library with several SC_TC_NPOLY values and sweep the wide windows.
set -x
OUT=gpurun_out/tcn
mkdir -p $OUT
for n in 0 16 24 32; do
  touch paper_2312_17649_b200/csrc/attn_tc.cu
  make -C paper_2312_17649_b200/csrc -j8 EXTRA=-DSC_TC_NPOLY=$n > $OUT/build_$n.log 2>&1
  echo "npoly=$n" >> $OUT/sweep.txt
  timeout 300 python scripts/attn_sweep.py --windows 128,256,inf >> $OUT/sweep.txt 2>&1
done
touch paper_2312_17649_b200/csrc/attn_tc.cu
make -C paper_2312_17649_b200/csrc -j8 > $OUT/build_default.log 2>&1
timeout 900 python -m pytest tests/test_gpu_attention.py -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
