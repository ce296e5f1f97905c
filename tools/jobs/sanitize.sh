# compute-sanitizer over the small decode runs of tools/sanitize_run.py
set -x
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 \
      python tools/sanitize_run.py > gpurun_out/r02_sanitize_$tool.log 2>&1
  echo "$tool rc=$?"
  tail -12 gpurun_out/r02_sanitize_$tool.log
done
