mkdir -p gpurun_out
./tools/lat_probe.bin > gpurun_out/lat_probe.txt 2>&1
timeout 300 python tools/probe_engines.py > gpurun_out/probe_engines.txt 2>&1
IT=50 ADMM_PERSIST_GRID=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:persist -s 1 -c 1 -o gpurun_out/full_persistgrid_q50 python tools/probe_persist.py > gpurun_out/ncu_full_persistgrid.log 2>&1
tail -3 gpurun_out/ncu_full_persistgrid.log
