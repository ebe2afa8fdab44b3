timeout 300 python tools/tmem_check.py --kernel tmem8 --configs c1,c2_3072x768,c4_2048x512_s80 2>&1 | tail -3
SDNN_TMEM_FILL=2 timeout 300 python tools/tmem_check.py --kernel tmem8 --configs c1,c2_3072x768,c4_2048x512_s80 2>&1 | tail -3
SDNN_TMEM_FILL=2 timeout 300 python tools/tmem_check.py --kernel tmem --configs c1,c4_2048x512_s80 2>&1 | tail -2
for f in 1 2; do SDNN_TMEM_FILL=$f timeout 200 python tools/time_cfg.py --config c5 --kernel tmem,tmem8 --iters 3 | sed "s/^/fill=$f /"; done
