mkdir -p gpurun_out/r01e
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/r01e/pytest_gpu.log 2>&1; tail -2 gpurun_out/r01e/pytest_gpu.log
p() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$1', '%.3e'%d['value'], r.get('kernel'), 'frac %.3f'%r['frac'], 'ms/launch %.4f'%r['avg_launch_ms'])"; }
for q in 10000 100000; do
  timeout 200 python bench.py --workload sweep --q $q --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r01e/bench_sweep_q$q.json 2>&1; p "cpt4 q$q" < gpurun_out/r01e/bench_sweep_q$q.json
  ADMM_SWEEP_CPT=2 timeout 200 python bench.py --workload sweep --q $q --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | p "cpt2 q$q"
  timeout 200 python bench.py --workload sweep --q $q --coeff-bits 32 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r01e/bench_sweep_q${q}_c32.json 2>&1; p "cpt4 c32 q$q" < gpurun_out/r01e/bench_sweep_q${q}_c32.json
done
