# metadata-format microbenchmark: MIO instruction count vs register-file bytes per nonzero
cd tools/microbench && nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o metafmt metafmt.cu && cd ../..
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/metafmt.log
timeout 300 tools/microbench/metafmt 2048 >> gpurun_out/metafmt.log 2>&1
cat gpurun_out/metafmt.log
