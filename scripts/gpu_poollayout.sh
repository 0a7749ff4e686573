mkdir -p gpurun_out
timeout 300 python scripts/pool_layout_probe.py > gpurun_out/pool_layout.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -m gpu --timeout 300 -p no:cacheprovider -k "pool or prefill or burst or predict_two or fullsize or closed or chunk" >> gpurun_out/pool_layout.log 2>&1
timeout 600 python bench.py --config c4 --sub c2 --steps 30 --warmup 5 --no-cpu > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
python -c "
import json; j=json.loads(open('gpurun_out/bench_c4.json').read().strip().splitlines()[-1])
print('C4', j['us_per_iteration'], j['roofline']['kernel_us'], j.get('burst_prefill'))
for k,s in j.get('sub_configs',{}).items(): print('SUB', k, s['us_per_iteration'], s['roofline']['kernel_us'], s.get('burst_prefill'))
" >> gpurun_out/pool_layout.log 2>&1
grep -v "^\.\|^$" gpurun_out/pool_layout.log | tail -14
