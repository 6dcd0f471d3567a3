python tools/probe_timing.py
ADMM_NO_GRAPH=1 python tools/probe_timing.py
ADMM_NO_GRAPH=1 ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active --clock-control none -k regex:sweep -s 100 -c 20 --csv python tools/probe_timing.py 2>&1 | grep -v "^==" | tail -90 > gpurun_out/ncu_sweep_q50.csv
Q=10000 ADMM_NO_GRAPH=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active --clock-control none -k regex:sweep -s 30 -c 5 --csv python tools/probe_timing.py 2>&1 | grep -v "^==" | tail -30 > gpurun_out/ncu_sweep_q1e4.csv
