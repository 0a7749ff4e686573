mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -q -m gpu -x --timeout 300 -p no:cacheprovider > gpurun_out/t_iter.log 2>&1; tail -3 gpurun_out/t_iter.log
timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
timeout 300 python scripts/trace_select.py 512,4096 > gpurun_out/trace_sel.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_iter.csv python scripts/microbench.py --iters 3 --sizes 64,512,4096 > /dev/null 2>&1
tail -2 gpurun_out/bench_q.err; cat gpurun_out/trace_sel.log | cut -c1-600
