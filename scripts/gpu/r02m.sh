set -x
mkdir -p gpurun_out
timeout -k 10 300 ./scripts/calib/stream > gpurun_out/r02m_stream.log 2>&1; cat gpurun_out/r02m_stream.log
timeout -k 10 300 python scripts/select_micro.py > gpurun_out/r02m_micro.log 2>&1; cat gpurun_out/r02m_micro.log
timeout -k 10 900 python bench.py --steps 100 --warmup 10 --no-cpu > gpurun_out/r02m_bench.json 2> gpurun_out/r02m_bench.err
python - <<'PY'
import json
j=json.load(open('gpurun_out/r02m_bench.json'))
print(j['us_per_iteration'], j['step_us']['median'], j['roofline']['kernel_us'])
for k,v in j['sub_configs'].items(): print(k, v['us_per_iteration'], v['roofline']['kernel_us'])
PY
