bash tools/jobs/r2_tune.sh
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -15
