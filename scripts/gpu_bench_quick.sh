mkdir -p gpurun_out
timeout 600 python bench.py --steps 100 --warmup 10 --cpu-seconds 3 > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; echo "bench exit $?"
TRAIL_SELECT=radix timeout 600 python bench.py --steps 100 --warmup 10 --no-cpu --no-burst > gpurun_out/bench_q_radix.json 2>> gpurun_out/bench_q.err
tail -3 gpurun_out/bench_q.err
