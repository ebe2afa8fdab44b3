timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for v in B C; do SDNN_PKG_DIR=ab/$v timeout 900 python tools/bench_configs.py --variants auto --graph > gpurun_out/v2_cfg_$v.jsonl 2> gpurun_out/v2_cfg_$v.err; done
for v in B C; do for shape in 4096x4096:0.9 2048x2048:0.9 1024x1024:0.9 1024x1024:0.7 512x512:0.7 2048x2048:0.7; do for n in 128 256 512 1000; do
  SDNN_PKG_DIR=ab/$v timeout 120 python tools/time_cfg.py --shape $shape --n $n --kernel auto --iters 20 | sed "s/^/$v /"
done; done; done
