timeout 900 python -m pytest tests -m gpu -q --timeout 600 2>&1 | tail -5
ncu --set full --import-source on --clock-control none -k regex:persist -s 1 -c 1 -o gpurun_out/persist_q50 python tools/probe_persist.py > gpurun_out/ncu_persist.log 2>&1
tail -3 gpurun_out/ncu_persist.log
