# compute-sanitizer over every kernel of libtrail.so at small shapes (scripts/sanitize.py)
set -x
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout -k 10 900 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 99 python scripts/sanitize.py > gpurun_out/r02_sanitize_$tool.log 2>&1
  echo "$tool exit $?" >> gpurun_out/r02_sanitize_$tool.log
  tail -4 gpurun_out/r02_sanitize_$tool.log
done
