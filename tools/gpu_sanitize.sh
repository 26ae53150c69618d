# compute-sanitizer over tools/sanitize_run.py -> gpurun_out/r02_sanitize_*.log
for t in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $t --print-limit 50 python tools/sanitize_run.py > gpurun_out/r02_sanitize_$t.log 2>&1
  echo "$t rc=$?"; tail -4 gpurun_out/r02_sanitize_$t.log
done
