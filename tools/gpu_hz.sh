timeout 300 python -m pytest tests/test_gpu_admm.py -q -x --timeout 60 -k "stream" 2>&1 | tail -1
for n in 100000 1000000; do for e in 0 1; do timeout 120 python -c "
import sys; sys.argv=['bench.py','--workload','horizon','--n','$n','--steps','3','--warmup','2','--no-cpu-baseline','--no-e2e']
" ; done; done
for n in 10000 100000 1000000; do timeout 200 python bench.py --workload horizon --n $n --steps 3 --warmup 2 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('horizon', $n, r['kernel'], '%.3e'%d['value'], 'frac %.3f'%r['frac'], 'it/s %.0f'%d['iterations_per_s'])"; done
