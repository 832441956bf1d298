# ncu --set full captures of the fast-path kernels (forward layer 0, and one backward layer)
mkdir -p gpurun_out
T=${1:-r2}
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_fast|k_hub|k_bin2|k_gs" -s 0 -c 4 -f -o gpurun_out/${T}_fwd \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-graph --profile-reps 0 > gpurun_out/${T}_fwd.log 2>&1; echo "full fwd rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_fast|k_hub|k_bin2|k_gs" -s 1040 -c 18 -f -o gpurun_out/${T}_bwd \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-graph --profile-reps 0 > gpurun_out/${T}_bwd.log 2>&1; echo "full bwd rc=$?"
