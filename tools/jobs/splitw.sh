for v in W16 W32; do for shape in 4096x4096:0.9 2048x2048:0.9 1024x1024:0.7 768x3072:0.9 512x4096:0.95 3072x768:0.9; do for n in 128 256 512; do
  SDNN_PKG_DIR=ab/$v timeout 120 python tools/time_cfg.py --shape $shape --n $n --kernel auto --iters 30 | sed "s/^/$v /"
done; done; done
