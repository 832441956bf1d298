mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
python -c "
import json; d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['phases_ms_last_step']); [print(k, round(v['ms'],4), round(v['frac_hbm'],3)) for k,v in d['kernels'].items()]"
tail -3 gpurun_out/bench.err
