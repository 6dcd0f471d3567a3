# synccheck with plain launches (ADMM_NO_GRAPH=1): isolates the conditional-graph artefact
D=gpurun_out/sanitize_r01; mkdir -p $D
for e in stream stream_rl stream_u4 stream_pf stream_rl_f32 stream_fx; do
  ADMM_NO_GRAPH=1 ENGINES=$e timeout 600 compute-sanitizer --tool synccheck --print-limit 4 --error-exitcode 9 python tools/sanitize_cases.py > $D/synccheck_nograph_$e.log 2>&1; echo "synccheck nograph $e rc=$? $(grep -E 'ERROR SUMMARY' $D/synccheck_nograph_$e.log | tail -1)"
done
ADMM_NO_GRAPH=1 ENGINES=stream_u4,stream_pf timeout 1500 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 10 --error-exitcode 9 python tools/sanitize_cases.py > $D/racecheck_u4_pf.log 2>&1; echo "racecheck u4/pf rc=$?"; grep -E "SUMMARY" $D/racecheck_u4_pf.log | tail -1
