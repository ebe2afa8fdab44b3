timeout 900 python -m pytest tests/test_gpu_conv.py -m gpu -q -x 2>&1 | tail -8
timeout 900 python tools/conv_bench.py --out gpurun_out/conv_bench.jsonl > gpurun_out/conv_bench.log 2>&1
