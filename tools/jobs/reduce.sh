timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_conv.py tests/test_gpu_guards.py tests/test_gpu_gather.py -m gpu -q -x -k "split or multi or guard or conv or gather" 2>&1 | tail -2
for shape in 768x3072:0.9 512x4096:0.9 256x2048:0.8; do timeout 120 python tools/time_cfg.py --shape $shape --n 128 --kernel auto --iters 30; done
timeout 120 python tools/time_cfg.py --config c2_768x768 --kernel row --iters 30
