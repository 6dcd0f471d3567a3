mkdir -p gpurun_out/cpt
export ADMM_SWEEP_CPT=4
Q=10000 IT=30 ENG=1 ADMM_NO_GRAPH=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:sweep_kernel -s 12 -c 1 -o gpurun_out/cpt/sweep_cpt4 python tools/probe_persist.py > gpurun_out/cpt/ncu.log 2>&1
v=sweep_cpt4
python tools/ncu_summary.py gpurun_out/cpt/$v.ncu-rep > gpurun_out/cpt/${v}_summary.txt 2>&1
python tools/ncu_lines.py gpurun_out/cpt/$v.ncu-rep 50 > gpurun_out/cpt/${v}_lines.txt 2>&1
python tools/ncu_inst_lines.py gpurun_out/cpt/$v.ncu-rep 60 > gpurun_out/cpt/${v}_inst.txt 2>&1
python tools/ncu_raw.py gpurun_out/cpt/$v.ncu-rep > gpurun_out/cpt/${v}_raw.txt 2>&1
ncu -i gpurun_out/cpt/$v.ncu-rep --page details --csv > gpurun_out/cpt/${v}_details.csv 2>&1
rm -f gpurun_out/cpt/*.ncu-rep
