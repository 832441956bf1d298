#!/bin/bash
# Round-2 pass: GPU tests, bench, small-kernel times, ncu --set full captures of the step's main kernels.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --no-depth-sweep > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_encoder|k_head" --csv --log-file gpurun_out/small.csv \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-graph --profile-reps 0 --no-depth-sweep > gpurun_out/small.log 2>&1; echo "small rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_fast|k_hub_rows|k_gs_tma" -s 0 -c 4 -f -o gpurun_out/prof_fwd \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-graph --profile-reps 0 --no-depth-sweep > gpurun_out/prof_fwd.log 2>&1; echo "full fwd rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_bin2|k_hub_seg|k_hub_fold|k_reduce" -s 200 -c 6 -f -o gpurun_out/prof_bwd \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-graph --profile-reps 0 --no-depth-sweep > gpurun_out/prof_bwd.log 2>&1; echo "full bwd rc=$?"
