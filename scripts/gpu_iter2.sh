mkdir -p gpurun_out; rm -f gpurun_out/iter.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 300 -p no:cacheprovider >> gpurun_out/iter.log 2>&1
timeout 600 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_sweep.py -q -m gpu -x --timeout 300 -p no:cacheprovider >> gpurun_out/iter.log 2>&1
cd scripts && timeout 300 python select_graph_micro.py 640,2048,4096,20480,81920 >> ../gpurun_out/iter.log 2>&1; cd ..
TRAIL_TRACE_SELECT=1 timeout 300 python scripts/trace_step.py 512 >> gpurun_out/iter.log 2>&1
timeout 600 python bench.py --config c4 --sub c2 --steps 30 --warmup 5 --no-cpu > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
python scripts/show_bench.py gpurun_out/bench_c4.json >> gpurun_out/iter.log 2>&1
python -c "
import json; j=json.loads(open('gpurun_out/bench_c4.json').read().strip().splitlines()[-1])
for s in j.get('sub_configs',[]): print('SUB', s['config']['workload'][:20], s['us_per_iteration'], s['roofline']['kernel_us'])
" >> gpurun_out/iter.log 2>&1
grep -E "passed|failed|FAIL|us per call|batch|value|SUB|roofline" gpurun_out/iter.log | tail -40
