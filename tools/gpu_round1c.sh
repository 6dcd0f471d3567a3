# round-1 evidence pass C (final kernels): tests, smoke, bench lines, launch list, ncu full captures
mkdir -p gpurun_out/r01c
timeout 900 python -m pytest tests -m gpu -q --timeout 200 > gpurun_out/r01c/pytest_gpu.log 2>&1; tail -2 gpurun_out/r01c/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 400 python bench.py --steps 10 --warmup 3 > gpurun_out/r01c/bench_default.json 2> gpurun_out/r01c/bench_default.err
timeout 120 python bench.py --workload toy --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r01c/bench_toy.json 2>&1
for q in 1000 10000 100000; do timeout 200 python bench.py --workload sweep --q $q --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r01c/bench_sweep_q$q.json 2>&1; done
for n in 10000 100000 1000000; do timeout 200 python bench.py --workload horizon --n $n --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/r01c/bench_horizon_n$n.json 2>&1; done
for f in C R; do timeout 200 python bench.py --workload microbench --family $f --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r01c/bench_micro_$f.json 2>&1; done
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r01c/bench_reference.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01c/launches_default.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-secondary > gpurun_out/r01c/ncu_launch.log 2>&1
IT=200 timeout 600 ncu --set full --import-source on --clock-control none -k regex:persist_cluster -s 1 -c 1 -o gpurun_out/r01c/full_cluster_q50 python tools/probe_persist.py > gpurun_out/r01c/ncu_cluster.log 2>&1
Q=10000 IT=30 ENG=1 ADMM_NO_GRAPH=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:sweep_kernel -s 12 -c 1 -o gpurun_out/r01c/full_sweep_q1e4 python tools/probe_persist.py > gpurun_out/r01c/ncu_sweep.log 2>&1
for f in C R; do timeout 600 ncu --set full --import-source on --clock-control none -k regex:quartic -s 2 -c 1 -o gpurun_out/r01c/full_quartic_$f python bench.py --workload microbench --family $f --steps 1 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/r01c/ncu_quartic_$f.log 2>&1; done
# summaries on the box; keep only the headline report (gpurun_out must stay < 64 MiB)
for r in full_cluster_q50 full_sweep_q1e4 full_quartic_C full_quartic_R; do
  python tools/ncu_summary.py gpurun_out/r01c/$r.ncu-rep > gpurun_out/r01c/${r}_summary.txt 2>&1
  python tools/ncu_lines.py gpurun_out/r01c/$r.ncu-rep 30 > gpurun_out/r01c/${r}_lines.txt 2>&1
  python tools/ncu_inst_lines.py gpurun_out/r01c/$r.ncu-rep 30 > gpurun_out/r01c/${r}_inst.txt 2>&1
  python tools/ncu_raw.py gpurun_out/r01c/$r.ncu-rep > gpurun_out/r01c/${r}_raw.txt 2>&1
done
rm -f gpurun_out/r01c/full_sweep_q1e4.ncu-rep gpurun_out/r01c/full_quartic_C.ncu-rep gpurun_out/r01c/full_quartic_R.ncu-rep
du -sh gpurun_out
