set -x
mkdir -p gpurun_out
timeout 900 python bench.py --steps 100 --warmup 10 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?" >> gpurun_out/bench.err
timeout 300 python bench.py --steps 50 --warmup 10 --no-graph --no-cpu > gpurun_out/bench_nograph.json 2>> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/ncu_bench.log 2>&1; echo "ncu1 exit $?" >> gpurun_out/ncu_bench.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:umma -s 20 -c 2 -o gpurun_out/prof_umma python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/ncu_full.log 2>&1; echo "ncu2 exit $?" >> gpurun_out/ncu_full.log
timeout 900 python -m pytest tests/test_gpu_dist.py -q -m gpu --timeout 300 --timeout-method=thread -p no:cacheprovider > gpurun_out/gpu_tests2.log 2>&1; echo "tests exit $?" >> gpurun_out/gpu_tests2.log
cat gpurun_out/bench.json; cat gpurun_out/bench_nograph.json; tail -3 gpurun_out/bench.err; tail -3 gpurun_out/gpu_tests2.log
