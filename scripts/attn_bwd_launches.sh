#!/bin/bash
# ncu launch list of one sc_attn_bwd call (last iteration) for the two fine-tuning shapes.
mkdir -p gpurun_out
for cfg in "--nseq 8 --doc-len 4086" "--nseq 64 --doc-len 164"; do
  tag=$(echo $cfg | tr -d ' -')
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/bwd_$tag.csv python scripts/attn_bwd_prof.py $cfg --iters 1 > /dev/null 2>&1
  python - gpurun_out/bwd_$tag.csv <<'PY'
import csv, sys, collections
rows = [r for r in csv.DictReader(open(sys.argv[1])) if r.get("Metric Name") == "gpu__time_duration.sum"]
seen = collections.OrderedDict()
for r in rows:
    seen.setdefault(r["Kernel Name"][:90], []).append(float(r["Metric Value"]))
print(sys.argv[1])
for k, v in seen.items():
    print(f"{len(v):3d} {v[-1]/1000 if max(v) > 1000 else v[-1]:9.1f} {k}")
PY
done
