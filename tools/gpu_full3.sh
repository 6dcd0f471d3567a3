mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 200 > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py > gpurun_out/bench_default.json 2>gpurun_out/bench_default.err; python -c "
import json; d=json.loads(open('gpurun_out/bench_default.json').read().strip().splitlines()[-1])
print(d['value'], d['roofline']['frac'], d['gpu_launches'], d['e2e']['value'], d['cpu_baseline']['value'])
s=d['secondary'][0]; print(s['workload'], s['value'], s['roofline']['frac'], s['gpu_launches'])"
