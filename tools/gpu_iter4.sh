mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; tail -8 gpurun_out/pytest_gpu.log
ADMM_SO=$PWD/tools/libadmm_prof.so timeout 300 python tools/probe_phase.py
timeout 300 python tools/probe_engines.py 2>&1 | grep -v "grid=1"
