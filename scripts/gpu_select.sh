mkdir -p gpurun_out; rm -f gpurun_out/select.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x --timeout 300 -p no:cacheprovider -k "select" >> gpurun_out/select.log 2>&1
timeout 600 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_sweep.py -q -m gpu -x --timeout 300 -p no:cacheprovider >> gpurun_out/select.log 2>&1
cd scripts && timeout 300 python select_graph_micro.py >> ../gpurun_out/select.log 2>&1; cd ..
timeout 600 python bench.py --config c4 --sub '' --steps 30 --warmup 5 --no-cpu > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
python scripts/show_bench.py gpurun_out/bench_c4.json >> gpurun_out/select.log 2>&1
tail -30 gpurun_out/select.log
