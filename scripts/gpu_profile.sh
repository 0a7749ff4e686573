# round-end evidence: full bench line, ncu launch list of the bench command, one ncu --set full
# capture of each product kernel (n = 512 decode step)
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench exit $?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/ncu_bench.log 2>&1; echo "ncu1 exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fused|rank|pool_chunk" -c 6 -o gpurun_out/prof_full python scripts/microbench.py --iters 1 --sizes 512 > gpurun_out/ncu_full.log 2>&1; echo "ncu2 exit $?"
tail -2 gpurun_out/bench_full.err
