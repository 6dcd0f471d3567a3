mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; tail -15 gpurun_out/pytest_gpu.log
ADMM_SO=$PWD/tools/libadmm_prof.so timeout 300 python tools/probe_phase.py
timeout 300 python tools/probe_engines.py 2>&1 | grep -v "grid=1"
for f in R C; do timeout 300 python bench.py --workload microbench --family $f --steps 10 --warmup 3 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('micro', '$f', d['value'], d['roofline']['frac'])"; done
timeout 300 python bench.py --workload sweep --q 10000 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('sweep 1e4', d['value'], d['roofline']['frac'])"
