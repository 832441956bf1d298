#!/bin/bash
# ncu capture of selected kernels on the c3 bench step (one GPU).
# Usage: bash tools/gpu_prof.sh <kernel-regex> <skip> <count> [outname]
set -u
mkdir -p gpurun_out
RE=${1:-k_fast}; SKIP=${2:-0}; CNT=${3:-3}; OUT=${4:-prof}
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:$RE -s $SKIP -c $CNT -f -o gpurun_out/$OUT \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-graph --profile-reps 0 > gpurun_out/$OUT.log 2>&1
echo "ncu rc=$?"
