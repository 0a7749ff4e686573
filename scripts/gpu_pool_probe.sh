mkdir -p gpurun_out; rm -f gpurun_out/pool_probe.log
for r in 0 2 1; do echo "copy_rows $r" >> gpurun_out/pool_probe.log; TRAIL_POOL_COPY_ROWS=$r timeout 300 python scripts/trace_pool.py >> gpurun_out/pool_probe.log 2>&1; done
cat gpurun_out/pool_probe.log
