# quick GPU iteration: fast-path parity tests, then the c3 bench (no CPU baseline)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_config_parity.py tests/test_gpu_fast.py tests/test_gpu_parity.py -m gpu -q -x -rf > gpurun_out/pytest_iter.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_iter.log
timeout 900 python bench.py --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['loss'], d['phases_ms_last_step']); [print(k, round(v['ms'],4), round(v['frac_hbm'],3), v.get('ms_per_block')) for k,v in d['kernels'].items()]"
tail -3 gpurun_out/bench.err
