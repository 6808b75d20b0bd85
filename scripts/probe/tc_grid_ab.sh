cd $GRAFT_REPO_ROOT
for cfg in "SC_TC_HEAD_FAST=0 SC_TC_L2PROMO=2" "SC_TC_HEAD_FAST=1 SC_TC_L2PROMO=2" "SC_TC_HEAD_FAST=1 SC_TC_L2PROMO=1" "SC_TC_HEAD_FAST=0 SC_TC_L2PROMO=1" "SC_TC_HEAD_FAST=1 SC_TC_L2PROMO=0"; do
  echo "== $cfg"; env $cfg SWEEP_TC_ONLY=1 timeout 300 python scripts/sweep_quick.py > gpurun_out/ab.jsonl 2>&1; python scripts/show_sweep.py gpurun_out/ab.jsonl | tail -6
done
env SC_TC_HEAD_FAST=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:tc_attn -c 2 python scripts/attn_one.py --w 64 --iters 2 2>&1 | grep -E "dram|duration"
