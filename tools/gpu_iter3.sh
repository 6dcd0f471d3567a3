mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; tail -25 gpurun_out/pytest_gpu.log
ADMM_SO=$PWD/tools/libadmm_prof.so timeout 300 python tools/probe_phase.py
for f in 0.4 0.5 0.6 0.7 0.8 1.0; do echo "frac $f"; ADMM_TILE0_FRAC=$f timeout 300 python tools/probe_engines.py 2>&1 | grep "persist grid=0"; done
