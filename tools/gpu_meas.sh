# measurement pass: Table-3 analogue, bench with the depth sweep, CPU linearity (+1 full-depth CPU step)
mkdir -p gpurun_out
timeout 900 python tools/table3.py --out gpurun_out/r2_table3.json > gpurun_out/table3.log 2>&1; echo "table3 rc=$?"; tail -c 1500 gpurun_out/r2_table3.json
timeout 900 python bench.py --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/bench_sweep.json 2> gpurun_out/bench_sweep.err; echo "bench rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/bench_sweep.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['peak_hbm_depth_sweep'])"
timeout 1500 python tools/cpu_linearity.py --config c3 --full --out gpurun_out/r2_cpu_linearity.json > gpurun_out/cpulin.log 2>&1; echo "cpulin rc=$?"; cat gpurun_out/r2_cpu_linearity.json
GSRC_LIB=scratch/libgsrcuda_vC.so timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-depth-sweep --steps 5 --warmup 3 > gpurun_out/ab_vC.json 2> gpurun_out/ab_vC.err
echo "== vC rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/ab_vC.json').read().strip().splitlines()[-1]); print(round(d['value'],4), d['phases_ms_last_step']); [print(k, round(v['ms'],4), round(v['frac_hbm'],3), [round(x,4) for x in (v.get('ms_per_block') or [])]) for k,v in d['kernels'].items()]"
