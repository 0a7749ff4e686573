# session baseline: every GPU test, smoke, the default bench line (c4 + c2/c1 sub-records)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/nvsmi.txt
timeout 1200 python -m pytest tests -q -m gpu --timeout 600 --timeout-method=thread -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 600 python bench.py --steps 50 --warmup 5 --cpu-seconds 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?" >> gpurun_out/bench.err
tail -n 15 gpurun_out/gpu_tests.log; tail -n 2 gpurun_out/smoke.log; tail -n 3 gpurun_out/bench.err
