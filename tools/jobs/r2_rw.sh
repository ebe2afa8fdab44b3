# rows per warp of the TMEM-R kernel (SDNN_TMEM_RW experiments), c5 full N
for rw in 10 9 8; do
  SDNN_TMEM_RW=$rw timeout 300 python tools/time_cfg.py --config c5 --kernel tmem --iters 5 2>&1 | sed "s/^/rw=$rw /"
done
timeout 300 python tools/time_cfg.py --config c4_2048x512_s80 --kernel tmem --iters 20 2>&1
timeout 300 python tools/time_cfg.py --config c4_512x2048_s95 --kernel tmem --iters 20 2>&1
