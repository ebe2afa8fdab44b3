python tools/prof_one.py --config c2_768x768 --kernel auto --launches 3 > gpurun_out/r2_c2_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/r2_c2_launches.csv python tools/prof_one.py --config c2_768x768 --kernel auto --launches 3 > gpurun_out/r2_c2_ncu.log 2>&1
for ks in 1 2 4 8; do SDNN_SPLIT_K=$ks timeout 100 python tools/time_cfg.py --config c2_768x768 --kernel auto --iters 50 | sed "s/^/ks=$ks /"; done
timeout 100 python tools/time_cfg.py --config c2_768x768 --kernel auto,row,tmem --iters 50 --opts split_rows=0
