# 4 cells per thread (ILP 4, 256-thread CTAs) vs 2: parity subset + bench
p() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$1', '%.3e'%d['value'], r.get('kernel'), 'frac %.3f'%r['frac'], 'ms/launch %.4f'%r['avg_launch_ms'])"; }
ADMM_SWEEP_CPT=4 timeout 600 python -m pytest tests/test_gpu_admm.py -m gpu -q -x --timeout 300 -k "stream and not tma" 2>&1 | tail -2
for q in 10000 100000; do
  ADMM_SWEEP_CPT=2 timeout 200 python bench.py --workload sweep --q $q --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | p "cpt2 q$q"
  for fx in 0 1; do
  ADMM_SWEEP_FX=$fx ADMM_SWEEP_CPT=4 timeout 200 python bench.py --workload sweep --q $q --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | p "cpt4 fx$fx q$q"
  done
done
