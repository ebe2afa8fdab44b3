for f in 1 2; do for d in 0 2; do SDNN_TMEM_FILL=$f SDNN_DEBUG_TMEM=$d timeout 120 python tools/time_cfg.py --config c5 --kernel tmem,tmem8 --n 65536 | sed "s/^/fill=$f /"; done; done
SDNN_TMEM_FILL=2 timeout 200 python tools/tmem_check.py --kernel tmem8 --configs c2_3072x768,c4_2048x512_s80,c4_512x2048_s95 --c5
SDNN_TMEM_FILL=2 timeout 200 python tools/tmem_check.py --kernel tmem --configs c4_2048x512_s80,c4_512x2048_s95
