mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 1800 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -12 gpurun_out/pytest_gpu.log
for q in 20 0; do
timeout 600 python tools/drift.py --config c3 --gemm tf32 --qshift $q --out gpurun_out/drift_c3_tf32_q$q.json > /dev/null 2>> gpurun_out/drift.err; echo "drift c3 q$q rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/drift_c3_tf32_q$q.json')); print(d['reconstruction'], d['mask_flip_rate']['mean'], d['mask_flip_rate']['max'], d['max_abs_activation'])"
done
timeout 1500 python tools/drift.py --config c5 --gemm tf32 --qshift 20 --stride 16 --lr-sweep 1e-4,3e-5,1e-5 --steps 6 --out gpurun_out/drift_c5_tf32_q20.json > /dev/null 2>> gpurun_out/drift.err; echo "drift c5 rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/drift_c5_tf32_q20.json')); print(d['reconstruction'], d['mask_flip_rate']['mean'], d['max_abs_activation'], d['lr_sweep'])"
timeout 900 python bench.py --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['loss'], d['phases_ms_last_step']); [print(k, round(v['ms'],4), round(v['frac_hbm'],3), v.get('ms_per_block')) for k,v in d['kernels'].items()]"
tail -3 gpurun_out/bench.err
