#!/bin/bash
# compute-sanitizer on the round-2 fast path (k_fws, k_bin2, hub pre-passes, side-stream dW reductions),
# then the GPU tests of the encoder/head kernels and their per-launch metrics.
set -u
mkdir -p gpurun_out
S=/usr/local/cuda/bin/compute-sanitizer
{
echo "## memcheck: test_fast_train_step[4-256-16-hubs1-0] (hub rows > 1024 edges, multi-chunk folds) and the deterministic step (graph capture, PDL, side streams)"
timeout 900 $S --tool memcheck python -m pytest -q -x "tests/test_gpu_fast.py::test_fast_train_step[4-256-16-hubs1-0]" tests/test_gpu_fast.py::test_fast_step_deterministic 2>&1 | grep -E "COMPUTE-SANITIZER|passed|failed|ERROR SUMMARY|Invalid|error" | head -20
echo "## racecheck (shared-memory hazards): test_fast_layer_forward_backward[4-256-16-1-False] and test_fast_train_step[4-256-16-hubs1-0]"
timeout 1200 $S --tool racecheck python -m pytest -q -x "tests/test_gpu_fast.py::test_fast_layer_forward_backward[4-256-16-1-False]" "tests/test_gpu_fast.py::test_fast_train_step[4-256-16-hubs1-0]" 2>&1 | grep -E "COMPUTE-SANITIZER|passed|failed|RACECHECK SUMMARY|hazard" | head -20
echo "## synccheck: test_fast_layer_forward_backward[4-256-16-1-False]"
timeout 900 $S --tool synccheck python -m pytest -q -x "tests/test_gpu_fast.py::test_fast_layer_forward_backward[4-256-16-1-False]" 2>&1 | grep -E "COMPUTE-SANITIZER|passed|failed|ERROR SUMMARY" | head -20
} > gpurun_out/sanitizers.txt 2>&1
echo "san done"; cat gpurun_out/sanitizers.txt | tail -12
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_config_parity.py -m gpu -q -x > gpurun_out/pytest_parity.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_parity.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_encoder|k_head" --csv --log-file gpurun_out/small.csv \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-graph --profile-reps 0 --no-depth-sweep > gpurun_out/small.log 2>&1; echo "small rc=$?"
