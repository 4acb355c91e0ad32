nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pipes2 tools/micro/pipes2.cu && /tmp/pipes2 > gpurun_out/pipes2.txt 2>&1
cat gpurun_out/pipes2.txt
