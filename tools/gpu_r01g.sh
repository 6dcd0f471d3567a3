# round-1 evidence pass g (row-loop sweep default, F2): tests, smoke, bench lines, launch list, ncu
set -x
D=gpurun_out/r01g; mkdir -p $D
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 > $D/pytest_gpu.log 2>&1; tail -1 $D/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $D/smoke.log 2>&1; tail -1 $D/smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 > $D/bench_default.json 2> $D/bench_default.err
timeout 120 python bench.py --workload toy --steps 10 --warmup 3 --no-cpu-baseline > $D/bench_toy.json 2>&1
for q in 1000 10000 100000; do timeout 300 python bench.py --workload sweep --q $q --steps 5 --warmup 3 --no-cpu-baseline > $D/bench_sweep_q$q.json 2>&1; done
for q in 10000 100000; do timeout 300 python bench.py --workload sweep --q $q --coeff-bits 32 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $D/bench_sweep_q${q}_c32.json 2>&1; done
for n in 10000 100000 1000000; do timeout 200 python bench.py --workload horizon --n $n --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > $D/bench_horizon_n$n.json 2>&1; done
for f in C R; do timeout 200 python bench.py --workload microbench --family $f --steps 10 --warmup 3 --no-cpu-baseline > $D/bench_micro_$f.json 2>&1; done
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > $D/bench_reference.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/launches_default.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-secondary > $D/ncu_launch.log 2>&1
python tools/launch_share.py $D/launches_default.csv > $D/launches_default_share.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/launches_sweep_q1e4.csv python bench.py --workload sweep --q 10000 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $D/ncu_launch2.log 2>&1
python tools/launch_share.py $D/launches_sweep_q1e4.csv > $D/launches_sweep_q1e4_share.txt 2>&1
Q=10000 IT=30 ENG=1 ADMM_NO_GRAPH=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:sweep_kernel -s 12 -c 1 -o $D/full_sweep_rl_q1e4 python tools/probe_persist.py > $D/ncu_sweep.log 2>&1
Q=100000 IT=20 ENG=1 ADMM_NO_GRAPH=1 timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:sweep_kernel -s 12 -c 1 --csv --log-file $D/dram_sweep_rl_q1e5.csv python tools/probe_persist.py > $D/ncu_sweep2.log 2>&1
IT=200 timeout 600 ncu --set full --import-source on --clock-control none -k regex:persist_cluster -s 1 -c 1 -o $D/full_cluster_q50 python tools/probe_persist.py > $D/ncu_cluster.log 2>&1
for r in full_sweep_rl_q1e4 full_cluster_q50; do
  python tools/ncu_summary.py $D/$r.ncu-rep > $D/${r}_summary.txt 2>&1
  python tools/ncu_lines.py $D/$r.ncu-rep 40 > $D/${r}_lines.txt 2>&1
  python tools/ncu_inst_lines.py $D/$r.ncu-rep 40 > $D/${r}_inst.txt 2>&1
  python tools/ncu_raw.py $D/$r.ncu-rep > $D/${r}_raw.txt 2>&1
done
rm -f $D/*.ncu-rep
du -sh gpurun_out
