# row scalars loaded with the item (no global round trip in the row finalisation)
p() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$1', '%.3e'%d['value'], r.get('kernel'), 'frac %.3f'%r['frac'], 'ms/launch %.4f'%r['avg_launch_ms'])"; }
timeout 900 python -m pytest tests/test_gpu_admm.py tests/test_f2_precision.py -m gpu -q -x --timeout 300 2>&1 | tail -2
for q in 10000 100000; do
  timeout 200 python bench.py --workload sweep --q $q --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | p "prod q$q"
  ADMM_SWEEP_FX=1 timeout 200 python bench.py --workload sweep --q $q --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | p "fx q$q"
  ADMM_SWEEP_PF=1 timeout 200 python bench.py --workload sweep --q $q --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | p "pf q$q"
  ADMM_SWEEP_CPT=4 timeout 200 python bench.py --workload sweep --q $q --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | p "cpt4 q$q"
done
timeout 200 python bench.py --workload horizon --n 1000000 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e | p "hz1e6"
