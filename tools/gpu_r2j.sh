#!/bin/bash
# Full GPU tests, the default bench line, and encoder/head per-launch metrics.
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 1200 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none -k regex:"k_encoder|k_head" --csv --log-file gpurun_out/small.csv \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-graph --profile-reps 0 --no-depth-sweep > gpurun_out/small.log 2>&1; echo "small rc=$?"
