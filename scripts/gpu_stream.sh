mkdir -p gpurun_out
cd scripts/calib && nvcc -gencode arch=compute_100a,code=sm_100a -O3 stream.cu -o stream && timeout 300 ./stream > ../../gpurun_out/stream.log 2>&1; cd ../..
cat gpurun_out/stream.log
