mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; tail -4 gpurun_out/pytest_gpu.log
Q=10000 IT=30 ENG=1 ADMM_NO_GRAPH=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:sweep_tma -s 12 -c 1 -o gpurun_out/full_sweeptma_q1e4 python tools/probe_persist.py > gpurun_out/ncu_tma.log 2>&1; tail -2 gpurun_out/ncu_tma.log
