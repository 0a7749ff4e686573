mkdir -p gpurun_out; rm -f gpurun_out/xpf.log
for cb in 0 8 16 4; do
  echo "xpf $cb" >> gpurun_out/xpf.log
  TRAIL_WIDE_XPF=$cb timeout 300 python scripts/wide_probe.py >> gpurun_out/xpf.log 2>&1
done
for cb in 0 8; do
  TRAIL_WIDE_XPF=$cb timeout 600 python bench.py --config c4 --sub '' --steps 30 --warmup 5 --no-cpu --no-burst > gpurun_out/bench_xpf$cb.json 2>/dev/null
  python -c "
import json; j=json.loads(open('gpurun_out/bench_xpf$cb.json').read().strip().splitlines()[-1])
print('C4 xpf $cb', j['us_per_iteration'], j['roofline']['kernel_us'])" >> gpurun_out/xpf.log 2>&1
done
timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -m gpu -x --timeout 300 -p no:cacheprovider >> gpurun_out/xpf.log 2>&1
cat gpurun_out/xpf.log
