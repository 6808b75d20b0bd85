#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over every attention kernel + the encoder loops.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out/sanitize
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool python scripts/sanitize_small.py > gpurun_out/sanitize/sanitizer_$tool.txt 2>&1
  echo "$tool rc=$?"; tail -2 gpurun_out/sanitize/sanitizer_$tool.txt
done
