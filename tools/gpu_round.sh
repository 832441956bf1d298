#!/bin/bash
# One GPU-box pass: parity tests, bench, launch list, ncu captures of the step's kernels.
# Usage (from this container): gpurun --timeout 3000 -- 'bash tools/gpu_round.sh [stages]'
set -u
mkdir -p gpurun_out
STAGES=${1:-"test smoke bench ref launches full"}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
for s in $STAGES; do
  case $s in
    test)
      timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log ;;
    smoke)
      timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log ;;
    bench)
      timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -c 600 gpurun_out/bench.json ;;
    benchfast)
      timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -c 600 gpurun_out/bench.json ;;
    configs)
      for c in c1 c2; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?"; done
      timeout 1200 python bench.py --config c5 --no-cpu-baseline --steps 2 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "bench c5 rc=$?" ;;
    ref)
      timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"; tail -c 300 gpurun_out/bench_ref.json ;;
    launches)
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches.csv \
        python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-graph --profile-reps 0 > gpurun_out/launches.log 2>&1; echo "launches rc=$?" ;;
    full)
      # forward: k_gs, hub pre-pass, FWD; backward: GS, hub, INV, hub(dense), BIN
      timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_fast|k_hub|k_bin2|k_gs" -s 0 -c 4 -f -o gpurun_out/prof_fwd \
        python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-graph --profile-reps 0 > gpurun_out/prof_fwd.log 2>&1; echo "full fwd rc=$?"
      timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_fast|k_hub|k_bin2|k_gs" -s 1040 -c 7 -f -o gpurun_out/prof_bwd \
        python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-graph --profile-reps 0 > gpurun_out/prof_bwd.log 2>&1; echo "full bwd rc=$?" ;;
  esac
done
