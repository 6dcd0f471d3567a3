p() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$1', '%.3e'%d['value'], r.get('kernel'), 'frac %.3f'%r['frac'], 'ms/launch %.4f'%r['avg_launch_ms'], 'it/s %.0f'%d['iterations_per_s'])"; }
for n in 100 1000 10000 100000; do
  timeout 200 python bench.py --workload horizon --n $n --steps 3 --warmup 2 --no-cpu-baseline --no-e2e | p "hz$n auto"
  ADMM_PERSIST_GRID=1 timeout 200 python bench.py --workload horizon --n $n --steps 3 --warmup 2 --no-cpu-baseline --no-e2e | p "hz$n grid"
  timeout 200 python bench.py --workload horizon --n $n --exec 1 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e | p "hz$n stream"
done
