python tools/prof_one.py --config c2_768x3072 --kernel row --launches 2 > gpurun_out/c2_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:spmm_tma -s 1 -c 1 -o gpurun_out/c2_row python tools/prof_one.py --config c2_768x3072 --kernel row --launches 2 > gpurun_out/c2_ncu.log 2>&1
