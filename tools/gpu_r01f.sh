mkdir -p gpurun_out/r01f
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/r01f/pytest_gpu.log 2>&1; tail -1 gpurun_out/r01f/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
p() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$1', '%.3e'%d['value'], r.get('kernel'), 'frac %.3f'%r['frac'], 'ms/launch %.4f'%r['avg_launch_ms'])"; }
for q in 1000 10000 100000; do timeout 200 python bench.py --workload sweep --q $q --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r01f/bench_sweep_q$q.json 2>&1; p "sweep q$q" < gpurun_out/r01f/bench_sweep_q$q.json; done
for q in 10000 100000; do timeout 200 python bench.py --workload sweep --q $q --coeff-bits 32 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r01f/bench_sweep_q${q}_c32.json 2>&1; p "sweep c32 q$q" < gpurun_out/r01f/bench_sweep_q${q}_c32.json; done
