# round-end evidence: GPU tests, smoke, bench lines (c2 default, c1, c4, reference arm), ncu
# launch list of the bench command, ncu --set full of the product kernels
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x --timeout 600 --timeout-method=thread -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench exit $?" >> gpurun_out/bench_full.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 300 python bench.py --config c1 --steps 100 --warmup 10 --cpu-seconds 5 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 600 python bench.py --config c4 --steps 20 --warmup 5 --cpu-seconds 5 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/ncu_bench.log 2>&1; echo "ncu1 exit $?" >> gpurun_out/ncu_bench.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fused|rank|pool" -c 8 -o gpurun_out/prof_full python bench.py --steps 2 --warmup 3 --no-cpu --no-graph > gpurun_out/ncu_full.log 2>&1; echo "ncu2 exit $?" >> gpurun_out/ncu_full.log
python scripts/ncu_summary.py gpurun_out/prof_full.ncu-rep > gpurun_out/ncu_full_summary.csv 2>&1
tail -n 2 gpurun_out/gpu_tests.log; for f in gpurun_out/smoke.log gpurun_out/bench_full.err gpurun_out/ncu_bench.log gpurun_out/ncu_full.log; do tail -n 1 "$f"; done; cat gpurun_out/bench_ref.json
