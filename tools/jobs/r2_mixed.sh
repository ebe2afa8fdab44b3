# mixed operand path microbenchmark: TMEM-ld warps + shared-memory warps concurrently
cd tools/microbench && nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o mixed mixed.cu && cd ../..
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/mixed.log
timeout 300 tools/microbench/mixed 2048 >> gpurun_out/mixed.log 2>&1
cat gpurun_out/mixed.log
