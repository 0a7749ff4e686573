set -x
mkdir -p gpurun_out
timeout -k 10 900 python bench.py --steps 200 --warmup 20 --no-cpu > gpurun_out/r02s_bench.json 2> gpurun_out/r02s_bench.err
python - <<'PY'
import json
j=json.load(open('gpurun_out/r02s_bench.json'))
print(j['us_per_iteration'], j['step_us']['median'], j['roofline']['kernel_us'], j['roofline']['frac'])
for k,v in j['sub_configs'].items(): print(k, v['us_per_iteration'], v['roofline']['kernel_us'], (v.get('burst_prefill') or {}).get('pool_frac_of_hbm'))
PY
timeout -k 10 300 python scripts/trace_pool.py > gpurun_out/r02s_trace_pool.log 2>&1; tail -1 gpurun_out/r02s_trace_pool.log
