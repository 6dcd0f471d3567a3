set -x
timeout 900 python -m pytest tests -m gpu -q --timeout 600 2>&1 | tail -30
timeout 600 python bench.py --steps 10 --warmup 3 2>&1 | tail -3
timeout 300 python bench.py --workload sweep --q 10000 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -2
timeout 300 python bench.py --workload microbench --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_phev.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_phev.log 2>&1
tail -3 gpurun_out/ncu_phev.log
