#!/bin/bash
# ncu --set full (with source) of one kernel on the c3 bench step. Usage: bash tools/gpu_ncu_kernel.sh <regex> <skip> <count> <out>
set -u
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$1" -s $2 -c $3 -f -o gpurun_out/$4 \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-graph --profile-reps 0 --no-depth-sweep > gpurun_out/$4.log 2>&1
echo "ncu rc=$?"
