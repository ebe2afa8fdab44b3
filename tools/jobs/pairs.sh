timeout 600 python -m pytest tests/test_gpu_conv.py tests/test_gpu_guards.py -m gpu -q 2>&1 | tail -2
SDNN_PKG_DIR=ab/PU timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "bitwise or config_parity or split or narrow" 2>&1 | tail -2
timeout 900 python tools/conv_bench.py --out gpurun_out/conv_bench7.jsonl > gpurun_out/conv_bench7.log 2>&1
for c in c2_768x768 c2_768x3072 c3_256x128 c1; do VARIANTS="A PU" CFG=$c KERN=row ITERS=30 bash tools/jobs/abn.sh; done
for shape in 4096x4096:0.9 768x3072:0.9; do for v in A PU; do SDNN_PKG_DIR=ab/$v timeout 120 python tools/time_cfg.py --shape $shape --n 128 --kernel auto --iters 30 | sed "s/^/$v /"; done; done
