set -x
mkdir -p gpurun_out
timeout -k 10 600 compute-sanitizer --tool memcheck --print-limit 20 python scripts/select_micro.py 20480 > gpurun_out/r02k_memcheck.log 2>&1; head -60 gpurun_out/r02k_memcheck.log
