for c in c2_3072x768 c3_512x512 c3_1024x512 c4_512x2048_s95 c4_2048x512_s95; do timeout 120 python tools/time_cfg.py --config $c --kernel auto,row,tmem --iters 30; done
for shape in 1024x1024:0.9 2048x2048:0.9 4096x1024:0.9; do for n in 1024 2048 4096; do timeout 120 python tools/time_cfg.py --shape $shape --n $n --kernel auto,row,tmem --iters 20; done; done
