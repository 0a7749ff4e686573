# ncu --set full of the c4 step kernels (K1b pool, K2d wide, K4b selection) and the c2 step
# kernels (K2c fused, K4 rank), one launch each after warm-up; eager launches (no graphs)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"wide|pool_bulk|bucket" -s 12 -c 7 -o gpurun_out/prof_c4 python bench.py --config c4 --sub '' --steps 3 --warmup 3 --no-cpu --no-graph --no-burst > gpurun_out/ncu_c4.log 2>&1; echo "ncu c4 exit $?" >> gpurun_out/ncu_c4.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fused|rank|pool" -s 9 -c 6 -o gpurun_out/prof_c2 python bench.py --config c2 --sub '' --steps 3 --warmup 3 --no-cpu --no-graph --no-burst > gpurun_out/ncu_c2.log 2>&1; echo "ncu c2 exit $?" >> gpurun_out/ncu_c2.log
tail -n 3 gpurun_out/ncu_c4.log gpurun_out/ncu_c2.log
