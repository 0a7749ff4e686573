mkdir -p gpurun_out
timeout 900 python bench.py --config c4 --steps 20 --warmup 5 --cpu-seconds 10 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "c4 exit $?"
timeout 300 python bench.py --config c1 --steps 100 --warmup 10 --cpu-seconds 5 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo "c1 exit $?"
tail -3 gpurun_out/bench_c4.err gpurun_out/bench_c1.err
