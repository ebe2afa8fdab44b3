timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "auto_takes or split_k or narrow" 2>&1 | grep -v "^$" | tail -30
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4
for v in A B; do for shape in 4096x4096:0.9 2048x2048:0.9 1024x1024:0.9 768x3072:0.9 512x4096:0.9; do for n in 128 256 512; do
  SDNN_PKG_DIR=ab/$v timeout 120 python tools/time_cfg.py --shape $shape --n $n --kernel auto --iters 20 | sed "s/^/$v /"
done; done; done
