# Round-1 evidence pass on one B200: GPU tests, smoke, bench lines, ncu launch
# list + full captures of the dominant kernels.  Outputs land in gpurun_out/.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_phev.json 2> gpurun_out/bench_phev.err; tail -c 3000 gpurun_out/bench_phev.json
timeout 300 python bench.py --workload toy --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_toy.json 2>&1
for q in 1000 10000 100000; do
  timeout 600 python bench.py --workload sweep --q $q --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_sweep_q$q.json 2>&1
done
for n in 10000 1000000; do
  timeout 600 python bench.py --workload horizon --n $n --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_horizon_n$n.json 2>&1
done
for f in R C; do
  timeout 600 python bench.py --workload microbench --family $f --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_micro_$f.json 2>&1
done
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.json 2>&1
# launch list of the default bench command (cold-cache, serialised: share, not absolute)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_phev.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_phev.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:sweep -c 40 --csv --log-file gpurun_out/launches_sweep_q1e4.csv \
  python bench.py --workload sweep --q 10000 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_sweep.log 2>&1
# full captures
timeout 900 ncu --set full --import-source on --clock-control none -k regex:persist -s 1 -c 1 -o gpurun_out/full_persist_q50 \
  python tools/probe_persist.py > gpurun_out/ncu_full_persist.log 2>&1
Q=10000 IT=30 ENG=1 ADMM_NO_GRAPH=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:sweep_kernel -s 12 -c 1 -o gpurun_out/full_sweep_q1e4 \
  python tools/probe_persist.py > gpurun_out/ncu_full_sweep.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:quartic -s 2 -c 1 -o gpurun_out/full_quartic_R \
  python bench.py --workload microbench --family R --steps 1 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_quartic.log 2>&1
ls -la gpurun_out
