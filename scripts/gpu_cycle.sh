# one build->measure cycle: parity tests, bench, launch list (+ optional full ncu capture)
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -q -m gpu -x --timeout 300 --timeout-method=thread -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/gpu_tests.log
TRAIL_SELECT=bitonic timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "select" --timeout 300 --timeout-method=thread -p no:cacheprovider > gpurun_out/gpu_tests_bitonic.log 2>&1; echo "tests exit $?" >> gpurun_out/gpu_tests_bitonic.log
timeout 600 python bench.py --steps 200 --warmup 20 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?" >> gpurun_out/bench.err
timeout 300 python scripts/microbench.py --sizes ${MICRO_SIZES:-64,512,4096} > gpurun_out/micro.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/ncu_bench.log 2>&1; echo "ncu1 exit $?" >> gpurun_out/ncu_bench.log
if [ -n "$NCU_K" ]; then timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$NCU_K" -c ${NCU_C:-3} -o gpurun_out/prof_cycle python scripts/microbench.py --iters 2 --sizes 512 > gpurun_out/ncu_full.log 2>&1; echo "ncu2 exit $?" >> gpurun_out/ncu_full.log; fi
tail -3 gpurun_out/gpu_tests.log; tail -2 gpurun_out/gpu_tests_bitonic.log; tail -2 gpurun_out/bench.err; cat gpurun_out/micro.log
