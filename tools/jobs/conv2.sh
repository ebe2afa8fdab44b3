timeout 900 python -m pytest tests/test_gpu_conv.py -m gpu -q -x 2>&1 | tail -8
SDNN_CONV_GATHER=1 timeout 900 python -m pytest tests/test_gpu_conv.py -m gpu -q -x 2>&1 | tail -3
timeout 900 python tools/conv_bench.py --out gpurun_out/conv_bench2.jsonl > gpurun_out/conv_bench2.log 2>&1
