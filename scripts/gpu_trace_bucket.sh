mkdir -p gpurun_out
timeout 300 python scripts/trace_bucket.py 20480,81920 > gpurun_out/trace_bucket.log 2>&1
cat gpurun_out/trace_bucket.log
