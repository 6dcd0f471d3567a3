mkdir -p gpurun_out
timeout 120 python -m pytest tests/test_gpu_admm.py -k "stream and toy" -x -q --timeout 60 2>&1 | tail -3
timeout 600 python -m pytest tests -m gpu -q -x --timeout 120 > gpurun_out/pytest_gpu.log 2>&1; tail -12 gpurun_out/pytest_gpu.log
for q in 1000 10000 100000; do timeout 120 python bench.py --workload sweep --q $q --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('sweep', $q, '%.3e'%d['value'], 'frac %.3f'%d['roofline']['frac'], 'ms/it %.4f'%d['roofline']['avg_launch_ms'])"; done
for n in 100000 1000000; do timeout 120 python bench.py --workload horizon --n $n --steps 3 --warmup 2 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('horizon', $n, '%.3e'%d['value'], 'frac %.3f'%d['roofline']['frac'], 'ms/it %.4f'%d['roofline']['avg_launch_ms'])"; done
