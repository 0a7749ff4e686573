mkdir -p gpurun_out; rm -f gpurun_out/tf32.log
for v in tf32 ffma tf32 ffma; do
TRAIL_FP32_L1=$v timeout 600 python bench.py --config c1 --sub '' --steps 200 --warmup 10 --no-cpu > gpurun_out/bench_c1_$v.json 2> gpurun_out/bench_c1.err
TRAIL_FP32_L1=$v python -c "
import json; j=json.loads(open('gpurun_out/bench_c1_$v.json').read().strip().splitlines()[-1])
print('C1 $v', j['us_per_iteration'], j['step_us'], j['config']['l1_kernel'], j['roofline']['kernel_us'])
" >> gpurun_out/tf32.log 2>&1
done
cat gpurun_out/tf32.log
