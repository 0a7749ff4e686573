set -x
mkdir -p gpurun_out
timeout -k 10 300 python scripts/select_micro.py > gpurun_out/r02n_micro.log 2>&1; cat gpurun_out/r02n_micro.log
timeout -k 10 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02n_launches_selmicro.csv python scripts/select_micro.py 20480,81920 > /dev/null 2>&1
timeout -k 10 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider --timeout 400 -k "select" > gpurun_out/r02n_tests.log 2>&1; tail -3 gpurun_out/r02n_tests.log
timeout -k 10 900 python bench.py --steps 100 --warmup 10 --no-cpu > gpurun_out/r02n_bench.json 2> gpurun_out/r02n_bench.err
python - <<'PY'
import json
j=json.load(open('gpurun_out/r02n_bench.json'))
print(j['us_per_iteration'], j['step_us']['median'], j['roofline']['kernel_us'])
for k,v in j['sub_configs'].items(): print(k, v['us_per_iteration'], v['roofline']['kernel_us'])
PY
