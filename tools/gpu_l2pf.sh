p() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$1', '%.3e'%d['value'], r.get('kernel'), 'frac %.3f'%r['frac'], 'ms/launch %.4f'%r['avg_launch_ms'])"; }
for q in 10000 100000; do
  ADMM_SWEEP_CPT=4 timeout 200 python bench.py --workload sweep --q $q --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | p "cpt4 l2pf q$q"
  ADMM_SWEEP_CPT=4 ADMM_SO=paper_1903_10041_b200/exp/nol2pf.so timeout 200 python bench.py --workload sweep --q $q --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | p "cpt4 nopf q$q"
  ADMM_SWEEP_CPT=4 timeout 200 python bench.py --workload sweep --q $q --coeff-bits 32 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | p "cpt4 l2pf c32 q$q"
  ADMM_SWEEP_FX=1 ADMM_SWEEP_CPT=4 timeout 200 python bench.py --workload sweep --q $q --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | p "cpt4 fx l2pf q$q"
done
