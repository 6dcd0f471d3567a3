ncu --replay-mode application --section SourceCounters --section WarpStateStats --section SchedulerStats --section SpeedOfLight --import-source on --clock-control none -k regex:persist_cluster -c 1 -o gpurun_out/cluster_q50 python tools/probe_persist.py > gpurun_out/ncu_cluster.log 2>&1
tail -2 gpurun_out/ncu_cluster.log
Q=10000 IT=30 ENG=1 ADMM_NO_GRAPH=1 ncu --set full --import-source on --clock-control none -k regex:sweep_kernel -s 12 -c 1 -o gpurun_out/sweep_q1e4 python tools/probe_persist.py > gpurun_out/ncu_sweep.log 2>&1
tail -2 gpurun_out/ncu_sweep.log
