#!/bin/bash
# Timing experiment (results are wrong with the switches set): what the hub pre-passes cost inside the real step.
set -u
mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu-baseline --no-depth-sweep --no-e2e --profile-reps 0 > gpurun_out/e0.json 2>/dev/null; echo "base rc=$?"
GSRC_EXP_SKIP_DHUB=1 timeout 600 python bench.py --no-cpu-baseline --no-depth-sweep --no-e2e --profile-reps 0 > gpurun_out/e1.json 2>/dev/null; echo "no dense hub rc=$?"
GSRC_EXP_SKIP_SHUB=1 timeout 600 python bench.py --no-cpu-baseline --no-depth-sweep --no-e2e --profile-reps 0 > gpurun_out/e2.json 2>/dev/null; echo "no sparse INV hub rc=$?"
for f in e0 e1 e2; do python -c "import json;d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]);print('$f', d['value'], d['phases_ms_last_step'])"; done
