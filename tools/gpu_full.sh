mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 200 > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
ADMM_SWEEP_FX=1 timeout 600 python -m pytest tests/test_gpu_admm.py -m gpu -q --timeout 120 -k stream 2>&1 | tail -1
