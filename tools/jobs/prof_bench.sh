# launch list of the bench command (metrics pass) + one full capture of the top kernel on a short c5 run
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/pb_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/pb_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/pb_ncu1.log 2>&1
python tools/prof_one.py --config c5 --kernel auto --n 65536 > gpurun_out/pb_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:spmm_tmem -s 1 -c 1 -o gpurun_out/pb_tmem_full python tools/prof_one.py --config c5 --kernel auto --n 65536 > gpurun_out/pb_ncu2.log 2>&1
