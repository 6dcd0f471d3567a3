# ceiling experiment: the sweep with Algorithm 1's trig branch replaced by a clamp (wrong results, timing only)
p() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$1', '%.3e'%d['value'], r.get('kernel'), 'frac %.3f'%r['frac'], 'ms/launch %.4f'%r['avg_launch_ms'])"; }
for q in 10000 100000; do
  for cpt in 2 4; do
    ADMM_SWEEP_CPT=$cpt ADMM_SO=paper_1903_10041_b200/exp/cheap.so timeout 200 python bench.py --workload sweep --q $q --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | p "cheap cpt$cpt q$q"
  done
  ADMM_SWEEP_FX=1 ADMM_SO=paper_1903_10041_b200/exp/cheap.so timeout 200 python bench.py --workload sweep --q $q --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | p "cheap fx q$q"
  ADMM_SWEEP_PF=1 ADMM_SO=paper_1903_10041_b200/exp/cheap.so timeout 200 python bench.py --workload sweep --q $q --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | p "cheap pf q$q"
done
