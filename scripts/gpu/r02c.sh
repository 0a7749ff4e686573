# round 2 (c): cluster selection + new parity tests + smoke + bench (progress on stderr)
set -x
mkdir -p gpurun_out
timeout -k 10 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02c_smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/r02c_smoke.log
timeout -k 10 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "select or zero_support or release_mid or multi_layer or closed_loop" -p no:cacheprovider > gpurun_out/r02c_tests.log 2>&1; echo "tests rc $?" >> gpurun_out/r02c_tests.log
timeout -k 10 450 python -m pytest tests/test_gpu_dist2.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r02c_dist2.log 2>&1; echo "dist2 rc $?" >> gpurun_out/r02c_dist2.log
timeout -k 10 900 python bench.py --steps 100 --warmup 10 > gpurun_out/r02c_bench.json 2> gpurun_out/r02c_bench.err; echo "bench rc $?" >> gpurun_out/r02c_bench.err
tail -2 gpurun_out/r02c_smoke.log; tail -4 gpurun_out/r02c_tests.log; tail -3 gpurun_out/r02c_dist2.log; tail -12 gpurun_out/r02c_bench.err
