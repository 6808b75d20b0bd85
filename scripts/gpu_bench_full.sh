#!/bin/bash
# Full default bench line (as the driver runs it) + the stand-alone quick sweep for comparison.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
echo "bench rc=$?" >> gpurun_out/bench_full.err
timeout 300 python scripts/sweep_quick.py > gpurun_out/sweep_after.jsonl 2>&1
