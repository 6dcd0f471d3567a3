# launch-bound experiment: 64-register sweep (2 CTAs/SM, spills) vs product 128-register
p() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$1', '%.3e'%d['value'], r.get('kernel'), 'frac %.3f'%r['frac'], 'ms/launch %.4f'%r['avg_launch_ms'])"; }
for q in 10000 100000; do
  for fx in 0 1; do
    ADMM_SWEEP_FX=$fx ADMM_SO=paper_1903_10041_b200/exp/lb1024.so timeout 200 python bench.py --workload sweep --q $q --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | p "lb1024 fx$fx q$q"
  done
done
