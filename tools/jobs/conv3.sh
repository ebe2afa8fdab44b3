timeout 900 python -m pytest tests/test_gpu_conv.py -m gpu -q -x 2>&1 | tail -3
timeout 900 python tools/conv_bench.py --out gpurun_out/conv_bench5.jsonl > gpurun_out/conv_bench5.log 2>&1
