# K2d load-path probes at configs[3] (TRAIL_WIDE_DIAG: 0 full, 1 no X, 2 no W1, 3 no loads)
mkdir -p gpurun_out; rm -f gpurun_out/wide_probe.log
for dg in 0 1 2 3; do
  TRAIL_WIDE_DIAG=$dg timeout 300 python scripts/wide_probe.py >> gpurun_out/wide_probe.log 2>&1
done
cat gpurun_out/wide_probe.log
