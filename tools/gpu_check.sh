#!/bin/bash
# Quick check: fast-path GPU tests, c3 bench, and per-launch metrics of the kernels matching a regex.
# Usage: bash tools/gpu_check.sh <kernel-regex> <skip> <count>
set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fast.py tests/test_gpu_config_parity.py -m gpu -q -x > gpurun_out/pytest_fast.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_fast.log
timeout 600 python bench.py --no-cpu-baseline --no-depth-sweep --no-e2e > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none -k regex:"${1:-k_bin2}" -s ${2:-4} -c ${3:-8} --csv --log-file gpurun_out/kern.csv \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-graph --profile-reps 0 --no-depth-sweep > gpurun_out/kern.log 2>&1; echo "ncu rc=$?"
