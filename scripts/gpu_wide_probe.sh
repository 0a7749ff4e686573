mkdir -p gpurun_out; rm -f gpurun_out/wide_probe.log
for dg in 0 4 3 7; do
  TRAIL_WIDE_DIAG=$dg timeout 300 python scripts/wide_probe.py >> gpurun_out/wide_probe.log 2>&1
done
cat gpurun_out/wide_probe.log
