mkdir -p gpurun_out; rm -f gpurun_out/sel5.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 300 -p no:cacheprovider -k "select" >> gpurun_out/sel5.log 2>&1
timeout 300 python scripts/trace_bucket.py 20480,81920 >> gpurun_out/sel5.log 2>&1
cd scripts && timeout 300 python select_graph_micro.py 4096,20480,81920 >> ../gpurun_out/sel5.log 2>&1; cd ..
grep -v "^\.\|^$" gpurun_out/sel5.log | tail -12
