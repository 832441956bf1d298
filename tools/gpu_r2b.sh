mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 1500 python -m pytest tests/test_gpu_config_parity.py tests/test_gpu_dp.py -m gpu -q -s -rA > gpurun_out/pytest_cfg.log 2>&1; echo "cfg rc=$?"; tail -22 gpurun_out/pytest_cfg.log
timeout 600 python tools/drift.py --config c3 --gemm tf32 --out gpurun_out/drift_c3_tf32.json > /dev/null 2> gpurun_out/drift.err; echo "drift c3 tf32 rc=$?"; cut -c1-600 gpurun_out/drift_c3_tf32.json
timeout 600 python tools/drift.py --config c3 --gemm fp32 --out gpurun_out/drift_c3_fp32.json > /dev/null 2>> gpurun_out/drift.err; echo "drift c3 fp32 rc=$?"; cut -c1-600 gpurun_out/drift_c3_fp32.json
timeout 600 python tools/drift.py --config c2 --gemm fp32 --out gpurun_out/drift_c2_fp32.json > /dev/null 2>> gpurun_out/drift.err; echo "drift c2 fp32 rc=$?"; cut -c1-600 gpurun_out/drift_c2_fp32.json
timeout 900 python bench.py --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['phases_ms_last_step']); [print(k, round(v['ms'],4), round(v['frac_hbm'],3), v.get('ms_per_block')) for k,v in d['kernels'].items()]"
tail -3 gpurun_out/bench.err
