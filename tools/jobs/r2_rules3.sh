bash tools/jobs/r2_tune.sh
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "split or tune or auto" 2>&1 | tail -3
