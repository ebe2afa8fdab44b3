# per-CTA fixed cost: same M, N, density; K (= chunks per CTA) varies
for K in 1024 2048 4096 8192; do
  SDNN_PKG_DIR=ab/A timeout 120 python tools/time_cfg.py --shape 4096x$K:0.9 --n 65536 --kernel tmem,tmem8 --iters 5
done
