set -x
mkdir -p gpurun_out
timeout -k 10 300 python scripts/select_micro.py > gpurun_out/r02f_micro.log 2>&1; cat gpurun_out/r02f_micro.log


timeout -k 10 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "select" -p no:cacheprovider --timeout 240 > gpurun_out/r02f_tests.log 2>&1; tail -5 gpurun_out/r02f_tests.log
