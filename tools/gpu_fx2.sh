timeout 400 python -m pytest tests/test_gpu_admm.py -q -x --timeout 60 -k "stream" 2>&1 | tail -1
ADMM_SWEEP_FX=1 timeout 400 python -m pytest tests/test_gpu_admm.py -q -x --timeout 60 -k "stream" 2>&1 | tail -1
for q in 10000 100000; do timeout 120 python bench.py --workload sweep --q $q --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('sweep', $q, '%.3e'%d['value'], 'frac %.3f'%r['frac'])"; done
timeout 120 python bench.py --workload horizon --n 1000000 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('horizon 1e6', r['kernel'], '%.3e'%d['value'], 'frac %.3f'%r['frac'])"
