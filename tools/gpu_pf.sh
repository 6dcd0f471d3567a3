# cp.async-prefetching sweep (ADMM_SWEEP_PF=1): parity subset + bench vs product
p() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$1', '%.3e'%d['value'], r.get('kernel'), 'frac %.3f'%r['frac'], 'ms/launch %.4f'%r['avg_launch_ms'])"; }
ADMM_SWEEP_PF=1 timeout 600 python -m pytest tests/test_gpu_admm.py tests/test_f2_precision.py -m gpu -q -x --timeout 300 -k "stream or full_size or fp32" 2>&1 | tail -3
for q in 10000 100000; do
  for pf in 0 1; do
    ADMM_SWEEP_PF=$pf timeout 200 python bench.py --workload sweep --q $q --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | p "pf$pf q$q"
  done
  ADMM_SWEEP_PF=1 timeout 200 python bench.py --workload sweep --q $q --coeff-bits 32 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | p "pf1 c32 q$q"
done
