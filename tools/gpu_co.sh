# concurrent backward sweep: correctness tests, then bench at several co-residency settings
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_rev_fast.py tests/test_gpu_config_parity.py tests/test_gpu_fast.py -m gpu -q -x -rf > gpurun_out/pytest_co.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_co.log
grep -E "^rev " gpurun_out/pytest_co.log | head; python -m pytest tests/test_gpu_rev_fast.py -m gpu -q -s 2>&1 | grep -E "^rev" | head -12
for co in 0 2,1 3,1 1,1; do
  GSRC_CO=$co timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 --profile-reps 0 > gpurun_out/co_$co.json 2> gpurun_out/co_$co.err
  echo "== co=$co rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/co_$co.json').read().strip().splitlines()[-1]); print(round(d['value'],4), d['phases_ms_last_step'], d['loss'])"
done
timeout 600 python bench.py --mode rev --no-cpu-baseline --no-e2e --steps 3 --warmup 3 --profile-reps 0 > gpurun_out/rev.json 2> gpurun_out/rev.err
echo "== rev rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/rev.json').read().strip().splitlines()[-1]); print(round(d['value'],4), d['phases_ms_last_step'], d['loss'], d['peak_hbm_bytes'])"
tail -2 gpurun_out/rev.err
