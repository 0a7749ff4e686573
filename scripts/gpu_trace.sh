mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "predict or graph or deterministic or agree or closed" --timeout 200 -p no:cacheprovider > gpurun_out/t3.log 2>&1; tail -3 gpurun_out/t3.log
timeout 300 python scripts/trace_fused.py --n 512 --splits 0,4,6,7,8 > gpurun_out/trace512d.log 2>&1
timeout 300 python scripts/trace_fused.py --n 4096 --splits 0 >> gpurun_out/trace512d.log 2>&1
timeout 300 python scripts/trace_fused.py --n 64 --splits 0 >> gpurun_out/trace512d.log 2>&1
cat gpurun_out/trace512d.log
