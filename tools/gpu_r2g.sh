#!/bin/bash
# Round-2 A/B pass: GPU tests, bench with and without the warp-specialised FWD/INV, small-kernel and k_fws launch times.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --no-depth-sweep > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
GSRC_NO_WS=1 timeout 600 python bench.py --no-cpu-baseline --no-depth-sweep --no-e2e > gpurun_out/bench_nows.json 2> gpurun_out/bench_nows.err; echo "bench nows rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none -c 1500 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-graph --profile-reps 0 --no-depth-sweep > gpurun_out/launches.log 2>&1; echo "launches rc=$?"
