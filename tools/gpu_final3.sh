D=gpurun_out/sanitize_r01b; mkdir -p $D
for e in stream_rl stream_rl_f32; do
  ADMM_NO_GRAPH=1 ENGINES=$e timeout 1200 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 4 --error-exitcode 9 python tools/sanitize_cases.py > $D/racecheck_nograph_$e.log 2>&1; echo "racecheck nograph $e rc=$? $(grep -E 'RACECHECK SUMMARY' $D/racecheck_nograph_$e.log | tail -1)"
  ADMM_NO_GRAPH=1 ENGINES=$e timeout 600 compute-sanitizer --tool synccheck --print-limit 4 --error-exitcode 9 python tools/sanitize_cases.py > $D/synccheck_nograph_$e.log 2>&1; echo "synccheck nograph $e rc=$? $(grep -E 'ERROR SUMMARY' $D/synccheck_nograph_$e.log | tail -1)"
done
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 > $D/pytest_gpu.log 2>&1; echo "pytest: $(tail -1 $D/pytest_gpu.log)"
p() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$1', '%.3e'%d['value'], r.get('kernel'), 'frac %.3f'%r['frac'])"; }
for q in 10000 100000; do timeout 200 python bench.py --workload sweep --q $q --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | p "sweep q$q"; done
timeout 200 python bench.py --workload horizon --n 1000000 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e | p "hz1e6"
