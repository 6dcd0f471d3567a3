# ncu --set full of one streaming sweep launch (PHEV q=1e4): product (128 regs) vs 64-register variant
mkdir -p gpurun_out/lb
Q=10000 IT=30 ENG=1 ADMM_NO_GRAPH=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:sweep_kernel -s 12 -c 1 -o gpurun_out/lb/sweep_prod python tools/probe_persist.py > gpurun_out/lb/ncu1.log 2>&1
Q=10000 IT=30 ENG=1 ADMM_NO_GRAPH=1 ADMM_SO=paper_1903_10041_b200/exp/lb1024.so timeout 600 ncu --set full --import-source on --clock-control none -k regex:sweep_kernel -s 12 -c 1 -o gpurun_out/lb/sweep_lb1024 python tools/probe_persist.py > gpurun_out/lb/ncu2.log 2>&1
for r in sweep_prod sweep_lb1024; do
  python tools/ncu_summary.py gpurun_out/lb/$r.ncu-rep > gpurun_out/lb/${r}_summary.txt 2>&1
  python tools/ncu_lines.py gpurun_out/lb/$r.ncu-rep 40 > gpurun_out/lb/${r}_lines.txt 2>&1
  python tools/ncu_inst_lines.py gpurun_out/lb/$r.ncu-rep 60 > gpurun_out/lb/${r}_inst.txt 2>&1
  python tools/ncu_raw.py gpurun_out/lb/$r.ncu-rep > gpurun_out/lb/${r}_raw.txt 2>&1
done

rm -f gpurun_out/lb/*.ncu-rep; du -sh gpurun_out
