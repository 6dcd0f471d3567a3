D=gpurun_out/r01i; mkdir -p $D
Q=10000 IT=30 ENG=1 ADMM_NO_GRAPH=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:sweep_kernel -s 12 -c 1 -o $D/full_sweep_rl_q1e4 python tools/probe_persist.py > $D/ncu_sweep.log 2>&1
r=full_sweep_rl_q1e4
python tools/ncu_summary.py $D/$r.ncu-rep > $D/${r}_summary.txt 2>&1
python tools/ncu_lines.py $D/$r.ncu-rep 40 > $D/${r}_lines.txt 2>&1
python tools/ncu_inst_lines.py $D/$r.ncu-rep 40 > $D/${r}_inst.txt 2>&1
python tools/ncu_raw.py $D/$r.ncu-rep > $D/${r}_raw.txt 2>&1
rm -f $D/*.ncu-rep
head -3 $D/${r}_raw.txt
