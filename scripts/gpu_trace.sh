mkdir -p gpurun_out
timeout 300 python scripts/trace_fused.py --n 512 --splits 0 > gpurun_out/trace_f.log 2>&1
cat gpurun_out/trace_f.log
