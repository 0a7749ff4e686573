set -x
mkdir -p gpurun_out
timeout -k 10 300 python scripts/select_micro.py > gpurun_out/r02i_micro.log 2>&1; cat gpurun_out/r02i_micro.log
timeout -k 10 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sweep.py tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider --timeout 400 -k "select or sweep or fullsize or closed" > gpurun_out/r02i_tests.log 2>&1; tail -5 gpurun_out/r02i_tests.log
timeout -k 10 900 python bench.py --steps 100 --warmup 10 > gpurun_out/r02i_bench.json 2> gpurun_out/r02i_bench.err; tail -3 gpurun_out/r02i_bench.err
python - <<'PY'
import json
j=json.load(open('gpurun_out/r02i_bench.json'))
print(j['us_per_iteration'], j['step_us']['median'], j['roofline']['kernel_us'])
for k,v in j['sub_configs'].items(): print(k, v['us_per_iteration'], v['roofline']['kernel_us'])
PY
timeout -k 10 300 python scripts/overlap.py --out gpurun_out/r02i_overlap.json > gpurun_out/r02i_overlap.log 2>&1; tail -2 gpurun_out/r02i_overlap.log
