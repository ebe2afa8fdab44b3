# A/B of two builds (ab/A, ab/B): parity of B, then c5 (N = 65536) and c4 80 % timings
SDNN_PKG_DIR=ab/B timeout 300 python tools/ab_parity.py 2>&1 | tail -14
for round in 1 2; do for v in A B; do
  SDNN_PKG_DIR=ab/$v timeout 200 python tools/time_cfg.py --config c5 --kernel tmem --iters 5 --n 65536 | sed "s/^/$v /"
  SDNN_PKG_DIR=ab/$v timeout 200 python tools/time_cfg.py --config c4_2048x512_s80 --kernel tmem --iters 20 | sed "s/^/$v /"
done; done
