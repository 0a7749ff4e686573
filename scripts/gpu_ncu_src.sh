mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fused|select" -c 4 -o gpurun_out/prof_src python scripts/microbench.py --iters 1 --sizes 512,4096 > gpurun_out/ncu_src.log 2>&1; echo "ncu exit $?"; tail -3 gpurun_out/ncu_src.log
