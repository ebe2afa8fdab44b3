timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
for v in A B; do for shape in 4096x4096:0.9 2048x2048:0.9 1024x1024:0.9 1024x1024:0.7 2048x2048:0.7 768x3072:0.9; do for n in 128 256 512 1024; do
  SDNN_PKG_DIR=ab/$v timeout 120 python tools/time_cfg.py --shape $shape --n $n --kernel auto --iters 20 | sed "s/^/$v /"
done; done; done
for v in A B; do SDNN_PKG_DIR=ab/$v timeout 900 python tools/bench_configs.py --variants auto --graph > gpurun_out/sk_cfg_$v.jsonl 2> gpurun_out/sk_cfg_$v.err; done
SDNN_PKG_DIR=ab/B timeout 1200 python tools/sweep.py --out gpurun_out/sweep4.jsonl > gpurun_out/sweep4.log 2>&1
