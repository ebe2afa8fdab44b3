timeout 300 python -m pytest tests/test_gpu_gather.py -q -x 2>&1 | tail -15
timeout 300 python bench.py --steps 3 --warmup 3 --allgather --no-cpu-baseline 2>&1 | tail -2
