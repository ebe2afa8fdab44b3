timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "narrow or config_parity or random or small or ragged or smoke" 2>&1 | tail -3
for v in C D; do for shape in 4096x4096:0.9 2048x2048:0.9 1024x1024:0.9 1024x1024:0.7 512x512:0.7 2048x2048:0.7; do for n in 128 256 512; do
  SDNN_PKG_DIR=ab/$v timeout 120 python tools/time_cfg.py --shape $shape --n $n --kernel auto --iters 20 | sed "s/^/$v /"
done; done; done
SDNN_PKG_DIR=ab/D timeout 1200 python tools/sweep.py --out gpurun_out/sweep3.jsonl > gpurun_out/sweep3.log 2>&1
