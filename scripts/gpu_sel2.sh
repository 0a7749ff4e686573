mkdir -p gpurun_out; rm -f gpurun_out/sel2.log
cd scripts && timeout 300 python select_graph_micro.py 640,2048,4096,20480,81920 >> ../gpurun_out/sel2.log 2>&1; cd ..
timeout 300 python scripts/trace_fused.py >> gpurun_out/sel2.log 2>&1
cat gpurun_out/sel2.log
