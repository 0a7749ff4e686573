mkdir -p gpurun_out; rm -f gpurun_out/wide_l2.log
for dg in 3 0; do TRAIL_WIDE_DIAG=$dg timeout 300 python scripts/wide_probe.py >> gpurun_out/wide_l2.log 2>&1; done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 120 -p no:cacheprovider -k "predict_two_steps or wide_tensor" >> gpurun_out/wide_l2.log 2>&1
timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -m gpu -x --timeout 300 -p no:cacheprovider >> gpurun_out/wide_l2.log 2>&1
grep -v "^\.\|^$" gpurun_out/wide_l2.log | tail -20
