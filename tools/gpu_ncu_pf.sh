mkdir -p gpurun_out/pf
for v in pf fx; do
  if [ $v = pf ]; then export ADMM_SWEEP_PF=1; unset ADMM_SWEEP_FX; else unset ADMM_SWEEP_PF; export ADMM_SWEEP_FX=1; fi
  Q=10000 IT=30 ENG=1 ADMM_NO_GRAPH=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:sweep_kernel -s 12 -c 1 -o gpurun_out/pf/sweep_$v python tools/probe_persist.py > gpurun_out/pf/ncu_$v.log 2>&1
  python tools/ncu_summary.py gpurun_out/pf/sweep_$v.ncu-rep > gpurun_out/pf/sweep_${v}_summary.txt 2>&1
  python tools/ncu_lines.py gpurun_out/pf/sweep_$v.ncu-rep 40 > gpurun_out/pf/sweep_${v}_lines.txt 2>&1
  python tools/ncu_inst_lines.py gpurun_out/pf/sweep_$v.ncu-rep 60 > gpurun_out/pf/sweep_${v}_inst.txt 2>&1
done
rm -f gpurun_out/pf/*.ncu-rep
