p() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$1', '%.3e'%d['value'], r.get('kernel'), 'frac %.3f'%r['frac'], 'ms/launch %.4f'%r['avg_launch_ms'])"; }
for bs in 512 256 128; do
  ADMM_SWEEP_BS=$bs timeout 200 python bench.py --workload horizon --n 1000000 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e | p "hz1e6 bs$bs"
done
for bs in 512 128; do
  ADMM_SWEEP_BS=$bs timeout 200 python bench.py --workload horizon --n 100000 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e | p "hz1e5 bs$bs"
done
