#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over scripts/sanitize_bwd.py -> gpurun_out/san_*.txt
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool python scripts/sanitize_bwd.py > gpurun_out/san_$tool.txt 2>&1
  tail -1 gpurun_out/san_$tool.txt
done
