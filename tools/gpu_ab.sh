# A/B: bench (per-class timings) + a short ncu launch list for each library variant
# usage: bash tools/gpu_ab.sh "name=path name=path ..."
mkdir -p gpurun_out
for nv in $1; do
  n=${nv%%=*}; p=${nv#*=}
  GSRC_LIB=$p timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 > gpurun_out/ab_$n.json 2> gpurun_out/ab_$n.err
  echo "== $n rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/ab_$n.json').read().strip().splitlines()[-1]); print(round(d['value'],4), d['phases_ms_last_step']); [print(k, round(v['ms'],4), round(v['frac_hbm'],3), [round(x,4) for x in (v.get('ms_per_block') or [])]) for k,v in d['kernels'].items()]"
  GSRC_LIB=$p timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_hub|k_fast|k_bin2|k_gs" -s 20 -c 60 --csv --log-file gpurun_out/ab_${n}_launch.csv \
     python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-graph --profile-reps 0 > /dev/null 2>&1
  python tools/ncu_summary.py launches gpurun_out/ab_${n}_launch.csv 2>/dev/null | head -14
done
