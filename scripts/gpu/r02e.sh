set -x
mkdir -p gpurun_out
timeout -k 10 300 python scripts/select_micro.py > gpurun_out/r02e_micro.log 2>&1
cat gpurun_out/r02e_micro.log
TRAIL_CSORT_ITEMS=8192 timeout -k 10 300 python scripts/select_micro.py 640,4096,20480,81920 > gpurun_out/r02e_micro8k.log 2>&1
cat gpurun_out/r02e_micro8k.log
timeout -k 10 600 ncu --set full --clock-control none --import-source on -k regex:select_cluster -c 4 -o gpurun_out/r02e_sel python scripts/select_micro.py 640,20480 > gpurun_out/r02e_ncu.log 2>&1; tail -3 gpurun_out/r02e_ncu.log
