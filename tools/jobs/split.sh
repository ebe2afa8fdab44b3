timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "split or bitwise or config_parity or desk or ragged or degenerate or host or graph" 2>&1 | tail -3
timeout 300 python tools/bench_configs.py --configs c2_768x768,c2_768x3072,c2_3072x768 --variants auto,row,tmem --graph --iters 10 2>/dev/null
