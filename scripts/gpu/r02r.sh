set -x
mkdir -p gpurun_out
timeout -k 10 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider --timeout 300 -k "prefill_start or pool or chunk or fullsize or two_steps" > gpurun_out/r02r_tests.log 2>&1; tail -3 gpurun_out/r02r_tests.log
timeout -k 10 600 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider --timeout 300 > gpurun_out/r02r_tests2.log 2>&1; tail -2 gpurun_out/r02r_tests2.log
timeout -k 10 900 python bench.py --steps 100 --warmup 10 --no-cpu > gpurun_out/r02r_bench.json 2> gpurun_out/r02r_bench.err; tail -2 gpurun_out/r02r_bench.err
python - <<'PY'
import json
j=json.load(open('gpurun_out/r02r_bench.json'))
print(j['us_per_iteration'], j['step_us']['median'], j['roofline']['kernel_us'])
for k,v in j['sub_configs'].items(): print(k, v['us_per_iteration'], v['roofline']['kernel_us'], (v.get('burst_prefill') or {}).get('pool_frac_of_hbm'))
PY
