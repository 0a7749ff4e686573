mkdir -p gpurun_out; rm -f gpurun_out/k2c.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 300 -p no:cacheprovider >> gpurun_out/k2c.log 2>&1
timeout 600 python bench.py --config c2 --sub '' --steps 200 --warmup 10 --no-cpu > gpurun_out/bench_c2.json 2>/dev/null
python -c "
import json; j=json.loads(open('gpurun_out/bench_c2.json').read().strip().splitlines()[-1])
print('C2', round(j['us_per_iteration'],2), j['step_us']['median'], j['roofline']['kernel_us'])
" >> gpurun_out/k2c.log 2>&1
grep -v "^\.\|^$" gpurun_out/k2c.log | tail -6
