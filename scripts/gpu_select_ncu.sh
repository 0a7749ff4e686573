mkdir -p gpurun_out
cd scripts && timeout 600 ncu --set full --clock-control none --import-source on -k regex:bucket -c 8 -o ../gpurun_out/prof_sel python select_graph_micro.py 20480,81920 > ../gpurun_out/ncu_sel.log 2>&1; echo "exit $?" >> ../gpurun_out/ncu_sel.log; cd ..
tail -3 gpurun_out/ncu_sel.log
