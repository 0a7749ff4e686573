mkdir -p gpurun_out
timeout 300 python scripts/pool_layout_probe.py > gpurun_out/pool_layout.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -m gpu --timeout 300 -p no:cacheprovider -k "pool or prefill or burst or predict_two or fullsize or closed or chunk" >> gpurun_out/pool_layout.log 2>&1
bash scripts/gpu_bench_quick2.sh >> gpurun_out/pool_layout.log 2>&1
grep -v "^\.\|^$" gpurun_out/pool_layout.log | tail -12
