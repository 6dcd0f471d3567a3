timeout 600 python -m pytest tests -m gpu -q -x --timeout 200 2>&1 | tail -1
timeout 120 python tools/probe_engines.py 2>&1 | grep "persist grid=0"
for q in 10000 100000; do timeout 120 python bench.py --workload sweep --q $q --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('sweep', $q, '%.3e'%d['value'], 'frac %.3f'%r['frac'])"; done
for f in R C; do timeout 120 python bench.py --workload microbench --family $f --steps 10 --warmup 3 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('micro $f', '%.3e'%d['value'], 'frac %.3f'%r['frac'])"; done
