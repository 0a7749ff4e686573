mkdir -p gpurun_out; rm -f gpurun_out/wmin.log
for wm in 2048 99999; do
TRAIL_WIDE_MIN=$wm timeout 900 python bench.py --sweep --sweep-n 2048,2560,3072,4096 --sweep-c 0.8 --no-cpu --sweep-out gpurun_out/wmin_$wm.json > /dev/null 2>&1
TRAIL_WIDE_MIN=$wm python -c "
import json; j=json.load(open('gpurun_out/wmin_$wm.json'))
for r in j['points']: print('$wm', r['n'], round(r['us_per_step_median'],1), r['l1_kernel'], r['kernel_us'])
" >> gpurun_out/wmin.log
done
cat gpurun_out/wmin.log
