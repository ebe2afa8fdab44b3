# ncu evidence for the cp-fill TMEM-R kernel: full capture (c5, N = 65536) and the bench launch list
python tools/prof_one.py --config c5 --kernel tmem --n 65536 --launches 2 > gpurun_out/r2_prof_plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:spmm_tmemr -s 1 -c 1 -o gpurun_out/r2_tmemr_cp_full python tools/prof_one.py --config c5 --kernel tmem --n 65536 --launches 2 > gpurun_out/r2_ncu3.log 2>&1
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-configs --no-proxy > gpurun_out/r2_bench_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_bench_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-configs --no-proxy > gpurun_out/r2_ncu_bench.log 2>&1
tail -2 gpurun_out/r2_ncu3.log gpurun_out/r2_ncu_bench.log
