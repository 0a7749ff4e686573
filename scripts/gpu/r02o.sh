set -x
mkdir -p gpurun_out
timeout -k 10 300 python scripts/trace_pool.py > gpurun_out/r02o_trace_pool.log 2>&1; tail -4 gpurun_out/r02o_trace_pool.log
timeout -k 10 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 > gpurun_out/r02o_tests.log 2>&1; tail -4 gpurun_out/r02o_tests.log
bash scripts/gpu/r02_sanitize.sh
