# ncu captures for round 2: pool (K1b) and K2d at configs[3], K2c and K4 at configs[1], the
# burst-prefill pool; plus the launch list (gpu__time_duration) of the default bench command
set -x
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-cpu"
timeout -k 10 900 ncu --set full --clock-control none --import-source on -k regex:"pool|wide" -c 4 -o gpurun_out/r02_ncu_c4 $B --sub "" > gpurun_out/r02_ncu_c4.log 2>&1; tail -2 gpurun_out/r02_ncu_c4.log
timeout -k 10 900 ncu --set full --clock-control none --import-source on -k regex:"fused|rank|pool" -c 6 -o gpurun_out/r02_ncu_c2 $B --config c2 --sub "" > gpurun_out/r02_ncu_c2.log 2>&1; tail -2 gpurun_out/r02_ncu_c2.log
timeout -k 10 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_launches_c4.csv $B --sub "" > gpurun_out/r02_launches_c4.log 2>&1; tail -2 gpurun_out/r02_launches_c4.log
timeout -k 10 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_selmicro.csv python scripts/select_micro.py 20480,81920 > gpurun_out/r02_launches_selmicro.log 2>&1; tail -1 gpurun_out/r02_launches_selmicro.log
