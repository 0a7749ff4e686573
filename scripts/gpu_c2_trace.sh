mkdir -p gpurun_out; rm -f gpurun_out/c2_trace.log
timeout 300 python scripts/wide_probe.py >> gpurun_out/c2_trace.log 2>&1
TRAIL_TRACE_SELECT=1 timeout 300 python scripts/trace_step.py 512 >> gpurun_out/c2_trace.log 2>&1
timeout 300 python scripts/trace_fused.py >> gpurun_out/c2_trace.log 2>&1
timeout 300 python scripts/graph_floor.py >> gpurun_out/c2_trace.log 2>&1
timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -m gpu -x --timeout 300 -p no:cacheprovider >> gpurun_out/c2_trace.log 2>&1
cat gpurun_out/c2_trace.log | tail -40
