set -x
mkdir -p gpurun_out
timeout -k 10 300 python scripts/trace_pool.py > gpurun_out/r02p_trace_pool.log 2>&1; tail -2 gpurun_out/r02p_trace_pool.log
timeout -k 10 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider --timeout 300 -k "pool or prefill or chunk or closed or layer" > gpurun_out/r02p_tests.log 2>&1; tail -3 gpurun_out/r02p_tests.log
timeout -k 10 900 python bench.py --steps 100 --warmup 10 --no-cpu > gpurun_out/r02p_bench.json 2> gpurun_out/r02p_bench.err
python - <<'PY'
import json
j=json.load(open('gpurun_out/r02p_bench.json'))
print(j['us_per_iteration'], j['step_us']['median'], j['roofline']['kernel_us'])
for k,v in j['sub_configs'].items(): print(k, v['us_per_iteration'], v['roofline']['kernel_us'], v.get('burst_prefill'))
PY
timeout -k 10 600 compute-sanitizer --tool racecheck --print-limit 10 python scripts/sanitize.py > gpurun_out/r02p_racecheck.log 2>&1; grep -v "Host Frame" gpurun_out/r02p_racecheck.log | tail -8
