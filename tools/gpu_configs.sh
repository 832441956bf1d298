#!/bin/bash
# The other BASELINE configs on one GPU: c1 (launch-bound), c2, and c5 (10M nodes, L = 200, C = 8).
# Usage (from this container): gpurun --timeout 2400 -- 'bash tools/gpu_configs.sh'
set -u
mkdir -p gpurun_out
for c in c1 c2; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-depth-sweep > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?"
done
timeout 1500 python bench.py --config c5 --no-cpu-baseline --no-depth-sweep --steps 2 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "bench c5 rc=$?"
