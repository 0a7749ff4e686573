# round-end evidence: GPU tests, smoke, bench lines (c4 default with c2/c1 sub-records,
# reference arm), ncu launch list of the bench command, ncu --set full of the product kernels
# per config (compute-sanitizer is closed on this pool: profiles/r02_sanitize_*.log are from
# earlier in the round)
mkdir -p gpurun_out/final
O=gpurun_out/final
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/nvsmi.txt
timeout 1500 python -m pytest tests -q -m gpu --timeout 600 --timeout-method=thread -p no:cacheprovider > $O/gpu_tests.log 2>&1; echo "tests exit $?" >> $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench exit $?" >> $O/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv --log-file $O/launches_bench.csv python bench.py --steps 5 --warmup 3 --no-cpu --no-burst > $O/ncu_launches.log 2>&1; echo "ncu launches exit $?" >> $O/ncu_launches.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"wide|pool_bulk|bucket" -s 14 -c 7 -o $O/prof_c4 python bench.py --config c4 --sub '' --steps 3 --warmup 3 --no-cpu --no-graph --no-burst > $O/ncu_c4.log 2>&1; echo "ncu c4 exit $?" >> $O/ncu_c4.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fused|rank|pool" -s 9 -c 6 -o $O/prof_c2 python bench.py --config c2 --sub '' --steps 3 --warmup 3 --no-cpu --no-graph --no-burst > $O/ncu_c2.log 2>&1; echo "ncu c2 exit $?" >> $O/ncu_c2.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gemv|head|rank" -s 9 -c 6 -o $O/prof_c1 python bench.py --config c1 --sub '' --steps 3 --warmup 3 --no-cpu --no-graph --no-burst > $O/ncu_c1.log 2>&1; echo "ncu c1 exit $?" >> $O/ncu_c1.log
TRAIL_FP32_L1=tf32 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"tf32" -s 3 -c 2 -o $O/prof_c1_tf32 python bench.py --config c1 --sub '' --steps 3 --warmup 3 --no-cpu --no-graph --no-burst > $O/ncu_c1_tf32.log 2>&1
for r in c4 c2 c1 c1_tf32; do python scripts/ncu_summary.py $O/prof_$r.ncu-rep > $O/ncu_${r}_summary.csv 2>&1; done
python scripts/launches.py $O/launches_bench.csv > $O/launches_bench_summary.txt 2>&1
tail -n 2 $O/gpu_tests.log; tail -n 1 $O/smoke.log $O/bench.err $O/ncu_launches.log $O/ncu_c4.log $O/ncu_c2.log $O/ncu_c1.log; cat $O/bench_reference.json
