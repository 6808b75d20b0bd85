set -x
mkdir -p gpurun_out/s2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/s2/smi.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/s2/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s2/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/s2/bench.json 2> gpurun_out/s2/bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/s2/bench_ref.json 2> gpurun_out/s2/bench_ref.err
timeout 600 python scripts/attn_sweep.py --windows 1,4,16,32,64,128,256,inf > gpurun_out/s2/sweep.jsonl 2>&1
timeout 600 python scripts/attn_sweep.py --windows inf --patterns full >> gpurun_out/s2/sweep.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s2/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/s2/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:band_attn -c 1 -o gpurun_out/s2/band_full python scripts/attn_sweep.py --windows 4 --iters 1 > gpurun_out/s2/ncu_band.log 2>&1
ls -la gpurun_out/s2
