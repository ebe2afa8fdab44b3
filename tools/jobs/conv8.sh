timeout 600 python -m pytest tests/test_gpu_conv.py tests/test_gpu_guards.py -m gpu -q 2>&1 | tail -2
timeout 900 python tools/conv_bench.py --out gpurun_out/conv_bench8.jsonl > gpurun_out/conv_bench8.log 2>&1
