mkdir -p gpurun_out
IT=100 timeout 600 ncu --set full --import-source on --clock-control none -k regex:persist_cluster -s 1 -c 1 -o gpurun_out/full_cluster_q50 python tools/probe_persist.py > gpurun_out/ncu_full_cluster.log 2>&1
tail -3 gpurun_out/ncu_full_cluster.log
IT=100 timeout 600 ncu --set full --import-source on --clock-control none -k regex:persist_cluster -s 1 -c 1 -o gpurun_out/full_cluster_toy python tools/probe_toy.py > gpurun_out/ncu_full_toy.log 2>&1
tail -3 gpurun_out/ncu_full_toy.log
