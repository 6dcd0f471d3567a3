# validation of HEAD: GPU suite, smoke, default bench, sweep/horizon lines
mkdir -p gpurun_out/r01d
timeout 900 python -m pytest tests -m gpu -q --timeout 200 > gpurun_out/r01d/pytest_gpu.log 2>&1; tail -2 gpurun_out/r01d/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 400 python bench.py --steps 10 --warmup 3 > gpurun_out/r01d/bench_default.json 2> gpurun_out/r01d/bench_default.err
for q in 10000 100000; do timeout 200 python bench.py --workload sweep --q $q --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r01d/bench_sweep_q$q.json 2>&1; done
timeout 200 python bench.py --workload horizon --n 1000000 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/r01d/bench_horizon_n1000000.json 2>&1
for f in gpurun_out/r01d/bench_*.json; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', '%.3e'%d['value'], d['roofline'].get('kernel'), 'frac %.3f'%d['roofline']['frac'])"; done
