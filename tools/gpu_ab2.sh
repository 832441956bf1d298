# A/B bench of library variants (per-class timings), then the dyadic/fast parity tests on the in-tree build
mkdir -p gpurun_out
for nv in $1; do
  n=${nv%%=*}; p=${nv#*=}
  GSRC_LIB=$p timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 > gpurun_out/ab_$n.json 2> gpurun_out/ab_$n.err
  echo "== $n rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/ab_$n.json').read().strip().splitlines()[-1]); print(round(d['value'],4), d['phases_ms_last_step']); [print(k, round(v['ms'],4), round(v['frac_hbm'],3), [round(x,4) for x in (v.get('ms_per_block') or [])]) for k,v in d['kernels'].items()]"
done
timeout 900 python -m pytest tests/test_gpu_config_parity.py tests/test_gpu_fast.py tests/test_gpu_rev_fast.py -m gpu -q -x -rf > gpurun_out/pytest_ab.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_ab.log
