# shorter-latency trig branch: latency probe old vs new, quartic + ADMM parity, benches
mkdir -p gpurun_out/trig
echo "--- old"; ./tools/lat_probe_old.bin | grep -E "boxmin|atan2|sincos|dfma"
echo "--- new"; ./tools/lat_probe.bin | grep -E "boxmin|atan2|sincos|dfma"
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/trig/pytest_gpu.log 2>&1; tail -2 gpurun_out/trig/pytest_gpu.log
p() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$1', '%.3e'%d['value'], r.get('kernel'), 'frac %.3f'%r['frac'], 'ms/launch %.4f'%r['avg_launch_ms'], 'it/s', d.get('iterations_per_s'))"; }
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/trig/bench_default.json 2>&1; p default < gpurun_out/trig/bench_default.json
for q in 10000 100000; do timeout 200 python bench.py --workload sweep --q $q --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/trig/bench_sweep_q$q.json 2>&1; p "sweep q$q" < gpurun_out/trig/bench_sweep_q$q.json; done
for q in 100000; do ADMM_SWEEP_CPT=4 timeout 200 python bench.py --workload sweep --q $q --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | p "sweep cpt4 q$q"; done
timeout 200 python bench.py --workload horizon --n 1000000 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/trig/bench_horizon_n1e6.json 2>&1; p "hz1e6" < gpurun_out/trig/bench_horizon_n1e6.json
for f in C R; do timeout 200 python bench.py --workload microbench --family $f --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/trig/bench_micro_$f.json 2>&1; p "micro $f" < gpurun_out/trig/bench_micro_$f.json; done
timeout 120 python bench.py --workload toy --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/trig/bench_toy.json 2>&1; p toy < gpurun_out/trig/bench_toy.json
