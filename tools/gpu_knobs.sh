# sweep-engine knob comparison (no rebuild): FX on/off, TMA engine
p() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$1', '%.3e'%d['value'], r.get('kernel'), 'frac %.3f'%r['frac'])"; }
for q in 10000 100000; do
  ADMM_SWEEP_FX=0 timeout 200 python bench.py --workload sweep --q $q --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | p "fx0 q$q"
  ADMM_SWEEP_FX=1 timeout 200 python bench.py --workload sweep --q $q --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | p "fx1 q$q"
  ADMM_STREAM_TMA=1 timeout 200 python bench.py --workload sweep --q $q --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | p "tma q$q"
done
