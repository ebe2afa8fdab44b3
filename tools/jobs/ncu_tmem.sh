python tools/prof_one.py --config c5 --kernel ${KERN:-tmem} --n 32768 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:spmm_tmem -s 1 -c 1 -o gpurun_out/tmem_c5 python tools/prof_one.py --config c5 --kernel ${KERN:-tmem} --n 32768 > gpurun_out/ncu_tmem.log 2>&1
