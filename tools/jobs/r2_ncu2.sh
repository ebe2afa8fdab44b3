python tools/prof_one.py --config c5 --kernel tmem --n 65536 --launches 2 > gpurun_out/r2_prof_plain.log 2>&1 && \
python tools/prof_one.py --config c4_512x2048_s95 --kernel auto --launches 2 >> gpurun_out/r2_prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:spmm_tmemr -s 1 -c 1 -o gpurun_out/r2_tmemr_full2 python tools/prof_one.py --config c5 --kernel tmem --n 65536 --launches 2 > gpurun_out/r2_ncu2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:spmm_ -s 1 -c 1 -o gpurun_out/r2_c4_95 python tools/prof_one.py --config c4_512x2048_s95 --kernel auto --launches 2 >> gpurun_out/r2_ncu2.log 2>&1
tail -3 gpurun_out/r2_ncu2.log
