mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x --timeout 300 -p no:cacheprovider > gpurun_out/t_iter.log 2>&1; tail -3 gpurun_out/t_iter.log
timeout 600 python bench.py --steps 100 --warmup 10 --no-cpu > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
TRAIL_PDL=0 timeout 600 python bench.py --steps 100 --warmup 10 --no-cpu --no-burst > gpurun_out/bench_q_nopdl.json 2>> gpurun_out/bench_q.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_iter.csv python scripts/microbench.py --iters 3 --sizes 64,512,4096 > /dev/null 2>&1
tail -2 gpurun_out/bench_q.err
