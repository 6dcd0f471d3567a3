ncu --set full --import-source on --clock-control none -k regex:persist_cluster -s 1 -c 1 -o gpurun_out/cluster_q50 python tools/probe_persist.py > gpurun_out/ncu_cluster.log 2>&1
tail -2 gpurun_out/ncu_cluster.log
