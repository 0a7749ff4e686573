set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r02a_gpu_tests.log
timeout 300 python bench.py > gpurun_out/r02a_bench_c2.json 2> gpurun_out/r02a_bench_c2.err
timeout 600 python bench.py --config c4 --steps 50 --warmup 5 > gpurun_out/r02a_bench_c4.json 2> gpurun_out/r02a_bench_c4.err
timeout 300 python bench.py --config c1 > gpurun_out/r02a_bench_c1.json 2> gpurun_out/r02a_bench_c1.err
tail -3 gpurun_out/r02a_gpu_tests.log; cat gpurun_out/r02a_bench_*.json | cut -c1-400
