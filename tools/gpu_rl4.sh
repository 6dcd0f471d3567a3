p() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$1', '%.3e'%d['value'], r.get('kernel'), 'frac %.3f'%r['frac'], 'ms/launch %.4f'%r['avg_launch_ms'])"; }
ADMM_SWEEP_RL_CPT=4 timeout 900 python -m pytest tests/test_gpu_admm.py -m gpu -q -x --timeout 300 -k "stream_rl" 2>&1 | tail -1
for q in 10000 100000; do
  timeout 200 python bench.py --workload sweep --q $q --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | p "rl2 q$q"
  ADMM_SWEEP_RL_CPT=4 timeout 200 python bench.py --workload sweep --q $q --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | p "rl4 q$q"
done
