mkdir -p gpurun_out; rm -f gpurun_out/trace_wide.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 120 -p no:cacheprovider -k "predict_two_steps or wide_tensor" >> gpurun_out/trace_wide.log 2>&1
timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -m gpu -x --timeout 300 -p no:cacheprovider >> gpurun_out/trace_wide.log 2>&1
timeout 300 python scripts/trace_wide.py >> gpurun_out/trace_wide.log 2>&1
timeout 300 python scripts/wide_probe.py >> gpurun_out/trace_wide.log 2>&1
grep -v "^\.\|^$" gpurun_out/trace_wide.log | tail -12
