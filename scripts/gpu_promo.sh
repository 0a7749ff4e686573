mkdir -p gpurun_out; rm -f gpurun_out/promo.log
for p in 3 2 1 0; do echo "promo $p" >> gpurun_out/promo.log; TRAIL_EMB_PROMO=$p timeout 300 python scripts/wide_probe.py >> gpurun_out/promo.log 2>&1; done
TRAIL_EMB_PROMO=0 TRAIL_WIDE_DIAG=2 timeout 300 python scripts/wide_probe.py >> gpurun_out/promo.log 2>&1
timeout 300 python scripts/trace_fused.py >> gpurun_out/promo.log 2>&1
cat gpurun_out/promo.log
