mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"pool" -c 4 -o gpurun_out/prof_pool python scripts/pool_probe.py 512 > gpurun_out/ncu_pool.log 2>&1; echo "ncu exit $?"; tail -2 gpurun_out/ncu_pool.log
