# round-1 evidence pass B: tests, default bench, launch list, full captures (profiles/)
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q --timeout 120 > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_phev.json 2> gpurun_out/bench_phev.err; cat gpurun_out/bench_phev.json
timeout 120 python bench.py --workload toy --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_toy.json 2>&1
for q in 1000 10000 100000; do timeout 200 python bench.py --workload sweep --q $q --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_sweep_q$q.json 2>&1; done
for n in 10000 100000 1000000; do timeout 200 python bench.py --workload horizon --n $n --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench_horizon_n$n.json 2>&1; done
for f in R C; do timeout 200 python bench.py --workload microbench --family $f --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_micro_$f.json 2>&1; done
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.json 2>&1
# launch list of the default bench command (cold-cache, serialised: compare shares)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_phev.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_phev.log 2>&1
# full captures of the dominant kernels
IT=200 timeout 600 ncu --set full --import-source on --clock-control none -k regex:persist_cluster -s 1 -c 1 -o gpurun_out/full_cluster_q50 python tools/probe_persist.py > gpurun_out/ncu_full_cluster.log 2>&1
Q=10000 IT=30 ENG=1 ADMM_NO_GRAPH=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:sweep_kernel -s 12 -c 1 -o gpurun_out/full_sweep_q1e4 python tools/probe_persist.py > gpurun_out/ncu_full_sweep.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:quartic -s 2 -c 1 -o gpurun_out/full_quartic_R python bench.py --workload microbench --family R --steps 1 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_quartic.log 2>&1
ls gpurun_out | wc -l
