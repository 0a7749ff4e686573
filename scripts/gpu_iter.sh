mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_parity.py -q -m gpu -x --timeout 300 -p no:cacheprovider > gpurun_out/t_iter.log 2>&1; tail -1 gpurun_out/t_iter.log
timeout 300 python bench.py --steps 200 --warmup 20 --no-cpu > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
timeout 300 python scripts/trace_fused.py --n 512 --splits 0 > gpurun_out/trace_f.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_iter.csv python bench.py --steps 5 --warmup 3 --no-cpu --no-burst > /dev/null 2>&1
tail -2 gpurun_out/bench_q.err
