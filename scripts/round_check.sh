#!/bin/bash
# Full GPU verification + measurement refresh: tests, smoke, bench (both arms), fine-tuning steps,
# attention-adjoint launch list.  Outputs under gpurun_out/check/.
set -u
O=gpurun_out/check
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.txt 2>&1
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
for a in "--doc-len 4086 --pairs 4" "--doc-len 164 --pairs 32"; do
  timeout 300 python scripts/train_bench.py $a >> $O/finetune.jsonl 2>> $O/finetune.err
  timeout 300 python scripts/train_bench.py $a --graph >> $O/finetune.jsonl 2>> $O/finetune.err
done
./scripts/attn_bwd_launches.sh > /dev/null 2>&1
python scripts/ncu_csv_summary.py gpurun_out/bwd_nseq*.csv > $O/attn_bwd_launches.txt
tail -1 $O/pytest_gpu.txt; tail -1 $O/smoke.txt; cat $O/bench.json | head -c 300; echo; cat $O/finetune.jsonl | cut -c1-200
