#!/bin/bash
# Usage (from this container): gpurun --timeout 3600 -- 'bash tools/gpu_round.sh'
# Evidence pass on one GPU box: full GPU tests, smoke, the default bench line (as the driver runs it), the reference arm,
# the launch list of one step and ncu --set full captures of the step's kernels.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-graph --profile-reps 0 --no-depth-sweep > gpurun_out/launches.log 2>&1; echo "launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_fws|k_hub|k_gs_tma" -s 0 -c 4 -f -o gpurun_out/prof_fwd \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-graph --profile-reps 0 --no-depth-sweep > gpurun_out/prof_fwd.log 2>&1; echo "full fwd rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_fws|k_hub|k_bin2|k_gs_tma|k_reduce" -s 1050 -c 8 -f -o gpurun_out/prof_bwd \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-graph --profile-reps 0 --no-depth-sweep > gpurun_out/prof_bwd.log 2>&1; echo "full bwd rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_encoder|k_head" --csv --log-file gpurun_out/small.csv \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-graph --profile-reps 0 --no-depth-sweep > gpurun_out/small.log 2>&1; echo "small rc=$?"
