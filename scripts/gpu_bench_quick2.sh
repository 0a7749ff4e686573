mkdir -p gpurun_out
timeout 900 python bench.py --steps 50 --warmup 5 --no-cpu > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
python -c "
import json; j=json.loads(open('gpurun_out/bench_q.json').read().strip().splitlines()[-1])
print('C4', round(j['us_per_iteration'],2), j['step_us']['median'], j['roofline']['frac'], j['roofline']['kernel_us'])
for k,s in j.get('sub_configs',{}).items(): print('SUB', k, round(s['us_per_iteration'],2), s['roofline']['kernel_us'])
"
