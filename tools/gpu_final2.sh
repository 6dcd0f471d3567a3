D=gpurun_out/sanitize_r01b; mkdir -p $D
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 > $D/pytest_gpu.log 2>&1; echo "pytest: $(tail -1 $D/pytest_gpu.log)"
for e in stream stream_rl stream_rl_f32; do
  ADMM_NO_GRAPH=1 ENGINES=$e timeout 1200 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 4 --error-exitcode 9 python tools/sanitize_cases.py > $D/racecheck_nograph_$e.log 2>&1; echo "racecheck nograph $e rc=$? $(grep -E 'RACECHECK SUMMARY' $D/racecheck_nograph_$e.log | tail -1)"
done
for e in stream_fx stream_u4; do
  ADMM_NO_GRAPH=1 ENGINES=$e timeout 1200 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 4 --error-exitcode 9 python tools/sanitize_cases.py > $D/racecheck_nograph_$e.log 2>&1; echo "racecheck nograph $e rc=$? $(grep -E 'RACECHECK SUMMARY' $D/racecheck_nograph_$e.log | tail -1)"
done
ADMM_NO_GRAPH=1 ENGINES=stream,stream_rl,stream_u4,stream_pf,stream_rl_f32,stream_fx,cluster,grid timeout 900 compute-sanitizer --tool memcheck --print-limit 10 --error-exitcode 9 python tools/sanitize_cases.py > $D/memcheck_nograph.log 2>&1; echo "memcheck nograph rc=$? $(grep -E 'ERROR SUMMARY' $D/memcheck_nograph.log | tail -1)"
