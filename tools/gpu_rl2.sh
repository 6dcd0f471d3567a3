p() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$1', '%.3e'%d['value'], r.get('kernel'), 'frac %.3f'%r['frac'], 'ms/launch %.4f'%r['avg_launch_ms'])"; }
timeout 900 python -m pytest tests/test_gpu_admm.py -m gpu -q -x --timeout 300 -k "stream" 2>&1 | tail -1
for q in 1000 10000 100000; do
  ADMM_SWEEP_RL=1 timeout 200 python bench.py --workload sweep --q $q --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | p "rl q$q"
  timeout 200 python bench.py --workload sweep --q $q --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | p "cpt4 q$q"
done
ADMM_SWEEP_RL=1 timeout 200 python bench.py --workload sweep --q 100000 --coeff-bits 32 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | p "rl c32 q1e5"
