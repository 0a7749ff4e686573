set -x
mkdir -p gpurun_out
timeout -k 10 300 python scripts/select_micro.py > gpurun_out/r02j_micro.log 2>&1; cat gpurun_out/r02j_micro.log
timeout -k 10 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sweep.py tests/test_gpu_fullsize.py tests/test_gpu_dist2.py -m gpu -q -p no:cacheprovider --timeout 400 -k "select or sweep or fullsize or closed or two_process" > gpurun_out/r02j_tests.log 2>&1; tail -5 gpurun_out/r02j_tests.log
timeout -k 10 900 python bench.py --steps 100 --warmup 10 > gpurun_out/r02j_bench.json 2> gpurun_out/r02j_bench.err; tail -2 gpurun_out/r02j_bench.err
python - <<'PY'
import json
j=json.load(open('gpurun_out/r02j_bench.json'))
print(j['us_per_iteration'], j['step_us']['median'], j['roofline']['kernel_us'])
for k,v in j['sub_configs'].items(): print(k, v['us_per_iteration'], v['roofline']['kernel_us'])
PY
