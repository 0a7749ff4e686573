mkdir -p gpurun_out; rm -f gpurun_out/wide_probe.log
for cfg in "0 0" "0 2" "0 1"; do
  set -- $cfg
  TRAIL_WIDE_DIAG=$2 timeout 300 python scripts/wide_probe.py >> gpurun_out/wide_probe.log 2>&1
done
timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -m gpu -x --timeout 300 -p no:cacheprovider >> gpurun_out/wide_probe.log 2>&1
cat gpurun_out/wide_probe.log | tail -20
