set -x
mkdir -p gpurun_out
timeout -k 10 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02h_smoke.log 2>&1; tail -1 gpurun_out/r02h_smoke.log
timeout -k 10 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 400 > gpurun_out/r02h_tests.log 2>&1; tail -12 gpurun_out/r02h_tests.log
timeout -k 10 600 python scripts/simulate.py --jobs 1500 --seeds 2 --grid --out gpurun_out/r02h_simulate.json > gpurun_out/r02h_simulate.log 2>&1; tail -5 gpurun_out/r02h_simulate.log
