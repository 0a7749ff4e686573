# full ncu capture of kernels matching $NCU_K in the microbench (eager launches, no graphs)
set -x
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$NCU_K" -c ${NCU_C:-3} -o gpurun_out/prof_$NCU_TAG python scripts/microbench.py --iters 2 --sizes ${NCU_SIZES:-512} > gpurun_out/ncu_$NCU_TAG.log 2>&1; echo "ncu exit $?" >> gpurun_out/ncu_$NCU_TAG.log
tail -3 gpurun_out/ncu_$NCU_TAG.log
