bash tools/jobs/ab.sh
SDNN_PKG_DIR=ab/B timeout 300 python tools/tmem_check.py --kernel tmem --configs c1,c2_768x768,c2_3072x768,c3_512x512,c4_2048x512_s80,c4_512x2048_s95
