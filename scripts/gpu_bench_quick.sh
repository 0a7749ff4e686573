mkdir -p gpurun_out
timeout 300 python bench.py --steps 200 --warmup 20 --no-cpu > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; echo "bench exit $?"
tail -2 gpurun_out/bench_q.err
