set -x
mkdir -p gpurun_out
timeout -k 10 2400 python bench.py --sweep --steps 30 --warmup 5 --cpu-seconds 3 --sweep-out gpurun_out/r02_sweep.json > gpurun_out/r02q_sweep.log 2>&1; tail -3 gpurun_out/r02q_sweep.log
timeout -k 10 1500 python -m pytest tests/test_gpu_sweep.py -m gpu -q -p no:cacheprovider --timeout 900 > gpurun_out/r02q_sweep_tests.log 2>&1; tail -3 gpurun_out/r02q_sweep_tests.log
timeout -k 10 600 python scripts/overlap.py --out gpurun_out/r02_overlap.json > gpurun_out/r02q_overlap.log 2>&1; tail -1 gpurun_out/r02q_overlap.log
