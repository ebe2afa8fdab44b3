SDNN_TMEM_FILL=4 timeout 200 python tools/tmem_check.py --kernel tmem8 --configs c1,c2_3072x768,c3_512x512,c4_2048x512_s80,c4_512x2048_s95 --c5
SDNN_TMEM_FILL=4 timeout 200 python tools/tmem_check.py --kernel tmem --configs c1,c2_3072x768,c4_2048x512_s80 --c5
for f in 1 4; do SDNN_TMEM_FILL=$f timeout 120 python tools/time_cfg.py --config c5 --kernel tmem,tmem8 | sed "s/^/fill=$f /"; done
SDNN_TMEM_FILL=4 SDNN_DEBUG_TMEM=2 timeout 120 python tools/time_cfg.py --config c5 --kernel tmem,tmem8 --n 65536 | sed "s/^/fill=4 /"
