cd tools/microbench/cg5
./run_cg5 r64w8.cubin 26365 65536 8 16 4 64 > ../../../gpurun_out/cg5_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -c 1 -o ../../../gpurun_out/cg5_r64w8 ./run_cg5 r64w8.cubin 26365 65536 8 16 4 64 > ../../../gpurun_out/cg5_ncu.log 2>&1
