mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke.log
timeout 1500 python -m pytest tests/test_gpu_config_parity.py -m gpu -q -s -rA > gpurun_out/pytest_cfg.log 2>&1; echo "cfg rc=$?"; tail -15 gpurun_out/pytest_cfg.log
