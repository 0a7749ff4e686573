# round 2 (b): new parity tests (2-process shard selection, release mid-prefill, zero-support
# priors), then the default bench line (configs[3] headline + c2/c1 sub-records)
set -x
timeout 900 python -m pytest tests/test_gpu_dist2.py tests/test_gpu_parity.py -m gpu -x -q -k "dist2 or two_process or release_mid or zero_support or closed_loop" 2>&1 | tail -15 > gpurun_out/r02b_gpu_tests.log
ls gpurun_out/parity_exemptions/
timeout 900 python bench.py > gpurun_out/r02b_bench.json 2> gpurun_out/r02b_bench.err
tail -3 gpurun_out/r02b_gpu_tests.log; cut -c1-300 gpurun_out/r02b_bench.json; tail -5 gpurun_out/r02b_bench.err
