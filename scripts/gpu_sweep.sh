mkdir -p gpurun_out
timeout 2400 python bench.py --sweep --sweep-out gpurun_out/r02_sweep.json > gpurun_out/sweep.log 2>&1; echo "sweep exit $?" >> gpurun_out/sweep.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 300 -p no:cacheprovider -k "wide_tensor" >> gpurun_out/sweep.log 2>&1
tail -5 gpurun_out/sweep.log
