# round 2 (d): after the head-fallback shuffle fix
set -x
mkdir -p gpurun_out
timeout -k 10 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02d_smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/r02d_smoke.log
tail -2 gpurun_out/r02d_smoke.log
timeout -k 10 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "select or zero_support or release_mid or multi_layer or closed_loop" -p no:cacheprovider --timeout 240 > gpurun_out/r02d_tests.log 2>&1; echo "tests rc $?" >> gpurun_out/r02d_tests.log
tail -4 gpurun_out/r02d_tests.log
timeout -k 10 450 python -m pytest tests/test_gpu_dist2.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r02d_dist2.log 2>&1; echo "dist2 rc $?" >> gpurun_out/r02d_dist2.log
tail -3 gpurun_out/r02d_dist2.log
timeout -k 10 900 python bench.py --steps 100 --warmup 10 > gpurun_out/r02d_bench.json 2> gpurun_out/r02d_bench.err; echo "bench rc $?" >> gpurun_out/r02d_bench.err
tail -12 gpurun_out/r02d_bench.err
