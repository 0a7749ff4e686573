mkdir -p gpurun_out
TRAIL_FUSED_SPLITS=1 timeout 300 python scripts/trace_step.py 512 2>&1 | tail -1
TRAIL_FUSED_SPLITS=2 timeout 300 python scripts/trace_step.py 512 2>&1 | tail -1
TRAIL_PDL=0 timeout 300 python scripts/trace_step.py 512 2>&1 | tail -1
