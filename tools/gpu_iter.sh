# quick GPU iteration: parity tests, engine timings, default bench line
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; tail -15 gpurun_out/pytest_gpu.log
timeout 300 python tools/probe_engines.py > gpurun_out/probe_engines.txt 2>&1; cat gpurun_out/probe_engines.txt
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_phev.json 2>&1; tail -c 1500 gpurun_out/bench_phev.json
