# F2: GPU suite (incl. fp32-coefficient parity) + fp32 vs fp64 sweep bench lines
mkdir -p gpurun_out/f2
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -x > gpurun_out/f2/pytest_gpu.log 2>&1; tail -3 gpurun_out/f2/pytest_gpu.log
p() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$1', '%.3e'%d['value'], r.get('kernel'), 'frac %.3f'%r['frac'], 'ms/launch %.4f'%r['avg_launch_ms'])"; }
for q in 10000 100000; do
  for b in 64 32; do
    timeout 200 python bench.py --workload sweep --q $q --coeff-bits $b --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/f2/bench_sweep_q${q}_c$b.json 2>&1; p "q$q c$b" < gpurun_out/f2/bench_sweep_q${q}_c$b.json
  done
done
timeout 200 python bench.py --workload horizon --n 1000000 --coeff-bits 32 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/f2/bench_horizon_n1e6_c32.json 2>&1; p "hz1e6 c32" < gpurun_out/f2/bench_horizon_n1e6_c32.json
