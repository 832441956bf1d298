#!/bin/bash
# One GPU-box pass: parity tests, bench, launch list, ncu capture of the top kernel.
# Usage (from this container): gpurun --timeout 2400 -- 'bash tools/gpu_round.sh [stages]'
set -u
mkdir -p gpurun_out
STAGES=${1:-"test bench launches full"}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
for s in $STAGES; do
  case $s in
    test)
      timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" ;;
    smoke)
      timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" ;;
    bench)
      timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -c 3000 gpurun_out/bench.json ;;
    benchfast)
      timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -c 3000 gpurun_out/bench.json ;;
    ref)
      timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"; cat gpurun_out/bench_ref.json ;;
    launches)
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches.csv \
        python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-graph --profile-reps 0 > gpurun_out/launches.log 2>&1; echo "launches rc=$?" ;;
    full)
      timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_tile -s 40 -c 3 -f -o gpurun_out/prof \
        python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-graph --profile-reps 0 > gpurun_out/prof.log 2>&1; echo "full rc=$?" ;;
  esac
done
