mkdir -p gpurun_out; rm -f gpurun_out/sel4.log
timeout 300 python scripts/trace_bucket.py 20480,81920 >> gpurun_out/sel4.log 2>&1
cd scripts && timeout 300 python select_graph_micro.py 640,2048,4096,20480,81920 >> ../gpurun_out/sel4.log 2>&1; cd ..
TRAIL_TRACE_SELECT=1 timeout 300 python scripts/trace_select.py 512 >> gpurun_out/sel4.log 2>&1
cat gpurun_out/sel4.log
