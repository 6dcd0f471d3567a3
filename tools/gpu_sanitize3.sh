# compute-sanitizer over the sweep layouts (row loop with its single barrier per row, staged
# four-cell slab, prefetch, F2) and the default engines; synccheck per engine
D=gpurun_out/sanitize_r01; mkdir -p $D
E=stream,stream_rl,stream_u4,stream_pf,stream_rl_f32,stream_fx,cluster,grid
ENGINES=$E timeout 900 compute-sanitizer --tool memcheck --print-limit 10 --error-exitcode 9 python tools/sanitize_cases.py > $D/memcheck.log 2>&1; echo "memcheck rc=$?"; grep -E "ERROR SUMMARY" $D/memcheck.log | tail -1
for e in stream stream_rl stream_u4 stream_pf stream_rl_f32 stream_fx cluster grid; do
  ENGINES=$e timeout 600 compute-sanitizer --tool synccheck --print-limit 4 --error-exitcode 9 python tools/sanitize_cases.py > $D/synccheck_$e.log 2>&1; echo "synccheck $e rc=$? $(grep -E 'ERROR SUMMARY' $D/synccheck_$e.log | tail -1)"
done
ENGINES=stream,stream_rl,stream_rl_f32,stream_fx timeout 1500 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 10 --error-exitcode 9 python tools/sanitize_cases.py > $D/racecheck.log 2>&1; echo "racecheck rc=$?"; grep -E "SUMMARY" $D/racecheck.log | tail -2
