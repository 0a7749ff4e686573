mkdir -p gpurun_out
timeout 500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -q -m gpu -x --timeout 300 -p no:cacheprovider > gpurun_out/t_iter.log 2>&1; tail -1 gpurun_out/t_iter.log
timeout 300 python bench.py --steps 200 --warmup 20 --no-cpu > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_iter.csv python scripts/microbench.py --iters 3 --sizes 512,4096 > /dev/null 2>&1
timeout 600 python bench.py --config c4 --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
tail -2 gpurun_out/bench_q.err; grep -E "FAIL|Error" gpurun_out/t_iter.log | head -5
