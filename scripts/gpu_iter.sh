# one iteration: parity tests, trace of the fused kernel, per-kernel launch list (ncu)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -q -m gpu -x --timeout 300 -p no:cacheprovider > gpurun_out/t_iter.log 2>&1; tail -3 gpurun_out/t_iter.log
timeout 300 python scripts/trace_fused.py --n 512 --splits 0 > gpurun_out/trace_iter.log 2>&1
timeout 300 python scripts/trace_fused.py --n 4096 --splits 0 >> gpurun_out/trace_iter.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_iter.csv python scripts/microbench.py --iters 3 --sizes 64,512,4096 > /dev/null 2>&1
timeout 300 python scripts/microbench.py --sizes 64,512,4096 > gpurun_out/micro_iter.log 2>&1
cat gpurun_out/micro_iter.log
