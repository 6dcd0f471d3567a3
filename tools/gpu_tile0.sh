p() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$1', '%.3e'%d['value'], r.get('kernel'), 'frac %.3f'%r['frac'], 'it/s %.0f'%d['iterations_per_s'])"; }
for f in 0.2 0.3 0.4 0.5 0.6; do
  ADMM_TILE0_FRAC=$f timeout 200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-secondary | p "frac0=$f"
done
