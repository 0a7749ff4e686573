set -x
mkdir -p gpurun_out
for f in "" "--write-flush"; do
timeout -k 10 600 python bench.py --config c2 --sub "" --steps 200 --warmup 20 --no-cpu $f > gpurun_out/r02t_c2$f.json 2> /dev/null
python -c "
import json
j=json.load(open('gpurun_out/r02t_c2$f.json'))
print('$f', j['us_per_iteration'], j['step_us']['median'], j['roofline']['kernel_us'])"
TRAIL_HEAD_SPIN=1 timeout -k 10 600 python bench.py --config c2 --sub "" --steps 200 --warmup 20 --no-cpu $f > gpurun_out/r02t_c2spin$f.json 2> /dev/null
python -c "
import json
j=json.load(open('gpurun_out/r02t_c2spin$f.json'))
print('spin $f', j['us_per_iteration'], j['step_us']['median'], j['roofline']['kernel_us'])"
done
