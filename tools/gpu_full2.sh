mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 200 > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_phev.json 2>&1; python -c "import json; d=json.loads(open('gpurun_out/bench_phev.json').read().strip().splitlines()[-1]); print(d['value'], d['iterations_per_s'], d['roofline']['frac'], d['gpu_launches'], d['e2e']['value'])"
