timeout 600 python -m pytest tests/test_gpu_guards.py -m gpu -q 2>&1 | tail -15
SDNN_CONV_GATHER=1 timeout 600 python -m pytest tests/test_gpu_guards.py -m gpu -q -k conv 2>&1 | tail -3
