mkdir -p gpurun_out; rm -f gpurun_out/head.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 300 -p no:cacheprovider -k "f32 or tf32 or l1-1 or 1-0.0 or 1-0.5 or unfused or 3-0" >> gpurun_out/head.log 2>&1
for v in ffma tf32; do
TRAIL_FP32_L1=$v timeout 600 python bench.py --config c1 --sub '' --steps 200 --warmup 10 --no-cpu > gpurun_out/bench_c1_$v.json 2> /dev/null
TRAIL_FP32_L1=$v python -c "
import json; j=json.loads(open('gpurun_out/bench_c1_$v.json').read().strip().splitlines()[-1])
print('C1 $v', round(j['us_per_iteration'],2), j['step_us']['median'], j['config']['l1_kernel'], j['roofline']['kernel_us'])
" >> gpurun_out/head.log 2>&1
done
grep -v "^\.\|^$" gpurun_out/head.log | tail
