set -x
mkdir -p gpurun_out
timeout -k 10 300 python scripts/select_micro.py > gpurun_out/r02g_micro.log 2>&1; cat gpurun_out/r02g_micro.log
TRAIL_SELECT=cluster timeout -k 10 300 python scripts/select_micro.py 640,20480 > gpurun_out/r02g_micro_cluster.log 2>&1; cat gpurun_out/r02g_micro_cluster.log
timeout -k 10 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02g_smoke.log 2>&1; tail -1 gpurun_out/r02g_smoke.log
timeout -k 10 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_dist2.py tests/test_gpu_dist.py -m gpu -q -p no:cacheprovider --timeout 300 > gpurun_out/r02g_tests.log 2>&1; tail -8 gpurun_out/r02g_tests.log
timeout -k 10 900 python bench.py --steps 100 --warmup 10 > gpurun_out/r02g_bench.json 2> gpurun_out/r02g_bench.err; tail -4 gpurun_out/r02g_bench.err
python - <<'PY'
import json
j=json.load(open('gpurun_out/r02g_bench.json'))
print(j['us_per_iteration'], j['roofline']['kernel_us'])
for k,v in j['sub_configs'].items(): print(k, v['us_per_iteration'], v['roofline']['kernel_us'])
PY
