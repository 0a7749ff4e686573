set -x
mkdir -p gpurun_out
timeout 600 python scripts/microbench.py > gpurun_out/micro.log 2>&1; echo "micro exit $?" >> gpurun_out/micro.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"trail_(pool|head|select)" -s 12 -c 3 -o gpurun_out/prof_small python scripts/microbench.py --iters 3 --sizes 512 > gpurun_out/ncu_small.log 2>&1; echo "ncu exit $?" >> gpurun_out/ncu_small.log
cat gpurun_out/micro.log
